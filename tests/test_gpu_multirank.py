"""Two and three real processes sharding one chain on the CUDA kernel (gloo
process group, every rank on cuda:0).  Byte-identical to the single-GPU
integration.  With the fused peer transport the ranks' kernels order their
edge tiles on the device with bounded waits; on one GPU the processes'
contexts are time-sliced, so a waiting CTA never blocks its neighbour's
progress -- and a neighbour that stops raises PeerTimeoutError."""

import datetime
import faulthandler
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from conftest import bits, collect  # noqa: E402


def _chain(s, seed, stiff=None):
    rng = np.random.default_rng(seed)
    m = rng.uniform(0.5, 2.0, s)
    C = rng.uniform(500.0, 2000.0, s)
    if stiff is not None:
        C[stiff] = 1e8
    return m, C, rng.standard_normal(s), rng.standard_normal(s)


def _port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, s, nsteps, T, stiff, transport, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    faulthandler.dump_traceback_later(180)  # a stuck rank shows where, before collect ends it
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        torch.cuda.set_device(0)
        from paper_1702_02207_b200 import sharded

        sh = sharded.ShardedChain(*_chain(s, 21, stiff), 1e-3, halo_steps=T,
                                  transport=transport)
        fb = sh.run(nsteps)
        x, v = sh.gather()
        sh.close()
        if rank == 0:
            q.put((fb, x.numpy(), v.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, s, nsteps, T, stiff=None, transport="nccl"):
    return collect(_worker, (world, _port(), s, nsteps, T, stiff, transport), world)


@pytest.mark.parametrize("world,T,transport", [(2, 32, "nccl"), (3, 16, "nccl"),
                                               (2, 32, "peer"), (3, 16, "peer")])
def test_processes_share_a_chain_bit_identically(world, T, transport):
    """transport="peer": CUDA IPC buffers and interprocess events between the
    processes; the tile kernel writes the neighbours' ghost zones itself."""
    from paper_1702_02207_b200 import batched

    s, n = 200_000, 97
    fb, x, v = _run(world, s, n, T, transport=transport)
    ref = batched.integrate_chains(*_chain(s, 21), 1e-3, n)
    assert fb == 0
    assert bits(x) == bits(ref.x[0].cpu().numpy()) and bits(v) == bits(ref.v[0].cpu().numpy())


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_processes_report_first_divergence(transport):
    from paper_1702_02207_b200 import batched

    s = 60_000
    fb, _, _ = _run(2, s, 300, 32, stiff=50_000, transport=transport)
    ref = batched.integrate_chains(*_chain(s, 21, 50_000), 1e-3, 300, check=False)
    assert fb > 0 and fb == int(ref.first_bad[0])


# random decompositions across real processes (a fixed example set by
# default; scripts/hypothesis_soak.sh with HYPOTHESIS_SOAK explores more)
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

_SOAK = int(os.environ.get("HYPOTHESIS_SOAK", "1"))


# every example spawns fresh processes (~4 s): the module's 300 s bound
# scales with the example count under a soak (a 50x soak ran into it: the
# timeout ended example 76, not a hang -- no stack dump was due)
@pytest.mark.timeout(max(300, 10 * 3 * _SOAK))
@settings(max_examples=3 * _SOAK, deadline=None, derandomize=_SOAK == 1,
          suppress_health_check=[HealthCheck.too_slow])
@given(world=st.integers(2, 3), s=st.integers(20_000, 150_000), T=st.integers(4, 40),
       nsteps=st.integers(1, 130), transport=st.sampled_from(["nccl", "peer"]))
def test_processes_random_decompositions(world, s, T, nsteps, transport):
    from paper_1702_02207_b200 import batched

    fb, x, v = _run(world, s, nsteps, T, transport=transport)
    ref = batched.integrate_chains(*_chain(s, 21), 1e-3, nsteps)
    assert fb == 0
    assert bits(x) == bits(ref.x[0].cpu().numpy()) and bits(v) == bits(ref.v[0].cpu().numpy())



def _worker_runs(rank, world, port, s, runs, T, transport, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    faulthandler.dump_traceback_later(180)  # a stuck rank shows where, before collect ends it
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        torch.cuda.set_device(0)
        from paper_1702_02207_b200 import sharded

        sh = sharded.ShardedChain(*_chain(s, 21), 1e-3, halo_steps=T, transport=transport)
        fb = 0
        for n in runs:
            fb = fb or sh.run(n)
        x, v = sh.gather()
        sh.close()
        if rank == 0:
            q.put((fb, x.numpy(), v.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_processes_several_runs_with_odd_periods(transport):
    """Consecutive run() calls of 3, 5 and 1 periods (the bench calls run()
    once per timed step) equal one run of the total steps, byte for byte."""
    from paper_1702_02207_b200 import batched

    s, T = 90_000, 16
    runs = (3 * T, 5 * T, T - 5)
    fb, x, v = collect(_worker_runs, (2, _port(), s, runs, T, transport), 2)
    ref = batched.integrate_chains(*_chain(s, 21), 1e-3, sum(runs))
    assert fb == 0
    assert bits(x) == bits(ref.x[0].cpu().numpy()) and bits(v) == bits(ref.v[0].cpu().numpy())


def test_peer_transport_host_ordering_fallback(monkeypatch):
    """Where stream waits on the mapped counters are unavailable, every rank
    orders periods on the host instead (OSC_PEER_HOST_ORDER=1 forces it):
    same bytes."""
    from paper_1702_02207_b200 import batched

    monkeypatch.setenv("OSC_PEER_HOST_ORDER", "1")
    s, T = 90_000, 16
    runs = (3 * T, T - 5)
    fb, x, v = collect(_worker_runs, (2, _port(), s, runs, T, "peer"), 2)
    ref = batched.integrate_chains(*_chain(s, 21), 1e-3, sum(runs))
    assert fb == 0
    assert bits(x) == bits(ref.x[0].cpu().numpy()) and bits(v) == bits(ref.v[0].cpu().numpy())


def _worker_stuck(rank, world, port, s, T, stuck, timeout_ms, q):
    """Rank `stuck` maps its buffers and counters but never runs a period;
    the others must get PeerTimeoutError instead of hanging."""
    import time

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    faulthandler.dump_traceback_later(180)  # a stuck rank shows where, before collect ends it
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        torch.cuda.set_device(0)
        from paper_1702_02207_b200 import sharded

        sh = sharded.ShardedChain(*_chain(s, 21), 1e-3, halo_steps=T, transport="peer",
                                  timeout_ms=timeout_ms)
        out = None
        if rank != stuck:
            t0 = time.monotonic()
            try:
                sh.run(6 * T)
                out = ("no error", None)
            except sharded.PeerTimeoutError as exc:
                out = ((exc.rank, exc.period, exc.side, exc.seen), time.monotonic() - t0)
        results = [None] * world
        dist.all_gather_object(results, out)
        sh.close()
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,stuck", [(2, 1), (3, 1)])
def test_stuck_neighbour_raises_instead_of_hanging(world, stuck):
    """The fused exchange's waits are bounded (osc_edge_sync_t.timeout_ns):
    a neighbour that never posts its edge counter makes every adjacent rank
    raise PeerTimeoutError naming itself, the period (1: period 0 needs only
    the initial state), the side and the counter value seen (0)."""
    results = collect(_worker_stuck, (world, _port(), 60_000, 8, stuck, 300.0), world)
    for rank, out in enumerate(results):
        if rank == stuck:
            assert out is None
            continue
        (r, period, side, seen), elapsed = out
        assert r == rank and period == 1 and seen == 0
        assert side == (1 if rank < stuck else 0)
        assert elapsed < 20.0  # one timeout, then the launches drain
