"""Multi-rank chain decomposition (BASELINE configs[2]) on CPU.

The ranks are real processes over torch.distributed (gloo, 127.0.0.1); the
per-shard advance is the oracle (the CUDA kernel needs a GPU -- the GPU tests
run the same driver with the kernel).  The result must be byte-identical to
the single-process integration for every rank count, as the reference's
engine is for every worker count (test_parallel.py:259-271)."""

import datetime
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
from conftest import bits, collect
from paper_1702_02207_b200 import sharded

pytestmark = pytest.mark.timeout(300)


def oracle_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0, first_bad,
                   tiles=None, **_):
    """Same contract as osc_rk4_chain_advance, on the CPU oracle: the buffer is
    treated as its own chain (wall at cell 0, free at n-1); only the owned
    cells are written and checked.  ``tiles``: "interior" writes only the
    owned cells farther than 2*nsteps cells from a ghost zone (they cannot
    depend on a ghost), "edges" the rest -- the contract of the OSC_TILES_*
    subsets (together one launch; the interior reads no ghost)."""
    x, v = xin.numpy().copy(), vin.numpy().copy()
    m, C = m.numpy(), C.numpy()
    for j in range(nsteps):
        with np.errstate(all="ignore"):
            x, v = oracle.np_rk4_step(m, C, x, v, dt)
        own = slice(own_lo, own_hi)
        if not (np.isfinite(x[own]).all() and np.isfinite(v[own]).all()):
            fb = int(first_bad.item())
            if fb == 0 or fb > step0 + j + 1:
                first_bad.fill_(step0 + j + 1)
            break
    n = xin.numel()
    keep = np.zeros(n, dtype=bool)
    keep[own_lo:own_hi] = True
    if tiles is not None:
        r = 2 * nsteps
        inner = np.zeros(n, dtype=bool)
        inner[own_lo + (r if own_lo > 0 else 0):own_hi - (r if own_hi < n else 0)] = True
        keep &= inner if tiles == "interior" else ~inner
    xout[keep] = torch.from_numpy(x[keep])
    vout[keep] = torch.from_numpy(v[keep])


def _chain(s, seed, stiff=None):
    rng = np.random.default_rng(seed)
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    if stiff is not None:
        C[stiff] = 1e8
    x0 = rng.standard_normal(s)
    v0 = rng.standard_normal(s)
    return m, C, x0, v0


def _free_port():
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def _worker(rank, world, port, s, nsteps, T, stiff, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        m, C, x0, v0 = _chain(s, 11, stiff)
        sh = sharded.ShardedChain(m, C, x0, v0, 1e-3, halo_steps=T, device=torch.device("cpu"),
                                  advance=oracle_advance)
        fb = sh.run(nsteps)
        x, v = sh.gather()
        if rank == 0:
            q.put((fb, x.numpy(), v.numpy()))
    finally:
        dist.destroy_process_group()


def _run_world(world, s, nsteps, T, stiff=None):
    return collect(_worker, (world, _free_port(), s, nsteps, T, stiff), world)


def test_layout():
    L = sharded.layout(100, 1, 4, 3)
    assert (L.lo, L.hi, L.blo, L.bhi, L.g) == (25, 50, 19, 56, 6)
    assert L.own == (6, 31) and L.n == 37
    L0 = sharded.layout(100, 0, 4, 3)
    assert L0.blo == 0 and L0.own == (0, 25)
    L3 = sharded.layout(100, 3, 4, 3)
    assert L3.bhi == 100 and L3.right_ghost == 0
    with pytest.raises(ValueError):
        sharded.layout(100, 0, 50, 3)


@pytest.mark.parametrize("world,T,nsteps", [(2, 8, 37), (3, 5, 40)])
def test_gloo_ranks_bit_identical(world, T, nsteps):
    s = 1500
    fb, x, v = _run_world(world, s, nsteps, T)
    m, C, x0, v0 = _chain(s, 11)
    _, _, xo, vo, fbo = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, nsteps,
                                            sample=False)
    assert fb == 0 and fbo[0] == 0
    assert bits(x) == bits(xo[0]) and bits(v) == bits(vo[0])


def test_gloo_divergence_is_min_over_ranks():
    s = 1500
    fb, _, _ = _run_world(3, s, 400, 8, stiff=1400)  # in the last rank's shard
    m, C, x0, v0 = _chain(s, 11, 1400)
    _, _, _, _, fbo = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, 400,
                                          sample=False)
    assert fbo[0] > 0 and fb == fbo[0]


def test_local_group_matches_single_chain():
    s = 3000
    m, C, x0, v0 = _chain(s, 5)
    grp = sharded.LocalShardGroup(m, C, x0, v0, 1e-3, 4, halo_steps=6,
                                  device=torch.device("cpu"), advance=oracle_advance)
    assert grp.run(45) == 0
    x, v = grp.gather()
    _, _, xo, vo, _ = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, 45,
                                          sample=False)
    assert bits(x.numpy()) == bits(xo[0]) and bits(v.numpy()) == bits(vo[0])


def peer_oracle_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0, first_bad,
                        left=None, right=None, **_):
    """oracle_advance plus the fused exchange: owned boundary cells are also
    written through the osc_peer_t descriptors (raw host pointers here)."""
    import ctypes

    oracle_advance(m, C, xin, vin, xout, vout, own_lo, own_hi, dt, nsteps, step0, first_bad)
    for side, desc in ((0, left), (1, right)):
        if desc is None:
            continue
        px, pv, offset, count = desc
        lo = own_lo if side == 0 else own_hi - count
        for ptr, src in ((px, xout), (pv, vout)):
            arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)),
                                        shape=(lo + count + offset,))
            arr[lo + offset:lo + count + offset] = src[lo:lo + count].numpy()


def test_local_group_peer_transport_matches_single_chain():
    s = 3000
    m, C, x0, v0 = _chain(s, 6)
    grp = sharded.LocalShardGroup(m, C, x0, v0, 1e-3, 4, halo_steps=6,
                                  device=torch.device("cpu"), advance=peer_oracle_advance,
                                  transport="peer")
    assert grp.run(45) == 0
    x, v = grp.gather()
    _, _, xo, vo, _ = oracle.c_rk4_chains(m[None], C[None], x0[None], v0[None], 1e-3, 45,
                                          sample=False)
    assert bits(x.numpy()) == bits(xo[0]) and bits(v.numpy()) == bits(vo[0])


def test_peer_descriptors_target_next_input_buffers():
    s = 400
    m, C, x0, v0 = _chain(s, 1)
    grp = sharded.LocalShardGroup(m, C, x0, v0, 1e-3, 2, halo_steps=4,
                                  device=torch.device("cpu"), transport="peer")
    a, b = grp.parts
    left, right = a.peer_descriptors(0)
    assert left is None
    # rank 0's last 8 owned cells land in rank 1's buffer 1 (its next input)
    assert right[0] == b.x2.data_ptr() and right[3] == 8
    assert right[2] == a.L.blo - b.L.blo
    l1, r1 = b.peer_descriptors(1)
    assert r1 is None and l1[0] == a.x.data_ptr()  # period 1: rank 0 reads buffer 1 next
