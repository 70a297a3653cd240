"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/osc_b200.h declares; the host API validates like the reference
and never falls back to the CPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1702_02207_b200 import _native
import paper_1702_02207_b200 as osc

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "osc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(osc_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        from paper_1702_02207_b200 import build

        build.build()
    return _native.load()


def test_header_declares_the_abi():
    syms = declared_symbols()
    for name in ("osc_rk4_batch2", "osc_rk4_chains", "osc_rk4_chain_advance",
                 "osc_rk4_batch2_host", "osc_rk4_chains_host", "osc_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert set(syms) == set(_native.SIGNATURES), "binding table out of sync with header"
    for name in syms:
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert lib.osc_abi_version() == _native.ABI_VERSION


def test_argument_errors_need_no_device(lib):
    # The reference's ValueError cases map to OSC_INVALID before any CUDA call.
    assert lib.osc_rk4_batch2(None, None, None, None, 4, float("nan"), 10, 1, None, None,
                              None, None, 0, None) == _native.OSC_INVALID
    assert b"dt must be positive" in lib.osc_last_error()
    assert lib.osc_rk4_batch2(None, None, None, None, 4, 1e-3, 0, 1, None, None, None,
                              None, 0, None) == _native.OSC_INVALID
    assert lib.osc_rk4_chains(None, None, None, None, 4, 3, 1e-3, 10, 0, None, None, None, None,
                              0, 0, None) == _native.OSC_INVALID
    assert b"stride" in lib.osc_last_error()
    # empty batch is a no-op success, as an empty loop would be
    assert lib.osc_rk4_batch2(None, None, None, None, 0, 1e-3, 10, 1, None, None, None,
                              None, 0, None) == _native.OSC_OK
    assert lib.osc_rk4_batch2(None, None, None, None, 4, 1e-3, 10, 1, None, None, None,
                              None, 0x80, None) == _native.OSC_INVALID
    assert b"flags" in lib.osc_last_error()
    assert lib.osc_rk4_chain_advance(None, None, None, None, None, None, 100, 0, 100, 1e-3, 600,
                                     0, None, None, None, None, 0, None) == _native.OSC_INVALID
    # validation entry points (modal.py): compare of an empty trajectory is
    # the reference's ValueError("empty trajectory") (modal.py:143-144)
    assert lib.osc_compare_batch2(None, None, None, 0, 4, None, None) == _native.OSC_INVALID
    assert b"empty trajectory" in lib.osc_last_error()
    assert lib.osc_compare_batch2(None, None, None, 3, 4, None, None) == _native.OSC_INVALID
    assert b"null buffer" in lib.osc_last_error()
    assert lib.osc_analytic_batch2(None, None, None, None, -1, None, None) == _native.OSC_INVALID
    assert lib.osc_analytic_batch2(None, None, None, None, 0, None, None) == _native.OSC_OK
    assert lib.osc_rk4_batch2_compare(None, None, None, None, 4, 1e-3, 10, 0, None, None, None,
                                      None, 0, None) == _native.OSC_INVALID
    assert b"stride" in lib.osc_last_error()
    assert lib.osc_rk4_batch2_compare(None, None, None, None, 4, 1e-3, 10, 1, None, None, None,
                                      None, 0, None) == _native.OSC_INVALID
    assert b"null buffer" in lib.osc_last_error()
    # single-process sharded chains validate before touching any device
    devs = (ctypes.c_int * 2)(0, 0)
    assert lib.osc_rk4_chain_sharded(0, devs, None, None, None, None, 100, 1e-3, 10, 0, None,
                                     0) == _native.OSC_INVALID
    assert lib.osc_rk4_chain_sharded(2, devs, None, None, None, None, 100, -1.0, 10, 0, None,
                                     0) == _native.OSC_INVALID
    assert lib.osc_rk4_chain_sharded(2, devs, None, None, None, None, 100, 1e-3, 10, 100, None,
                                     0) == _native.OSC_INVALID
    # dense and engine paths check shapes before touching the device
    assert lib.osc_rk4_dense(None, None, None, 0, 4, 1e-3, 10, None, None) == _native.OSC_INVALID
    assert lib.osc_rk4_dense(None, None, None, 8, 4, -1e-3, 10, None, None) == _native.OSC_INVALID
    assert lib.osc_equation_engine(None, None, None, None, 65, 1e-3, 10, 1, None, None, None,
                                   None, None) == _native.OSC_INVALID


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    system = osc.build_chain([1.0, 1.0], [1.0, 1.0])
    with pytest.raises(osc.NativeUnavailableError):
        osc.integrate(system, osc.PhaseState((1.0, 0.0), (0.0, 0.0)), 1e-3, 10)


def test_validation_mirrors_reference():
    with pytest.raises(osc.NonPositiveParameterError):
        osc.build_chain([1, -1], [1, 1])
    with pytest.raises(osc.NonPositiveParameterError):
        osc.build_chain([], [])
    with pytest.raises(osc.NonPositiveParameterError):
        osc.build_chain([float("nan")], [1])
    with pytest.raises(osc.LengthMismatchError):
        osc.build_chain([1, 1], [1])
    with pytest.raises(osc.NonFiniteStateError):
        osc.PhaseState((float("inf"),), (0.0,))
    system = osc.build_chain([0.002, 0.002], [20250, 20250])
    state = osc.PhaseState((2.0, -3.0), (0.0, 0.0))
    # integrate's checks come before any device work (oscillator.py:247-251)
    with pytest.raises(ValueError):
        osc.integrate(system, state, 1e-6, 0, 1)
    with pytest.raises(ValueError):
        osc.integrate(system, state, 1e-6, 10, 0)
    with pytest.raises(osc.LengthMismatchError):
        osc.integrate(system, osc.PhaseState((1.0,), (0.0,)), 1e-6, 10)
    for dt in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            osc.rk4_step(system, state, dt)


def test_accumulated_time_labels():
    from paper_1702_02207_b200.oscillator import accumulated_times

    t = 0.0
    ref = [t]
    for k in range(1, 2501):
        t += 1e-4
        if k % 7 == 0:
            ref.append(t)
    got = accumulated_times(0.0, 1e-4, 2500, 7)
    assert np.array(ref).tobytes() == got.tobytes()
    # chunk boundaries of the accumulation do not change the fold
    got = accumulated_times(1.5, 0.25, 3, 1)
    assert got.tolist() == [1.5, 1.75, 2.0, 2.25]


def test_workloads_are_seeded():
    from paper_1702_02207_b200 import workloads

    a = workloads.c2(B=1000)
    b = workloads.c2(B=1000)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    m, C, x0, v0 = a
    assert m.shape == (2, 1000) and (m >= 0.5).all() and (m < 2).all()
    assert (C >= 500).all() and (C < 2000).all() and not v0.any()
    # the multi-GPU split is a partition of the one draw (strong scaling)
    parts = [workloads.part(1000, r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate([m[:, p] for p in parts], axis=1), m)
    assert [p.stop - p.start for p in parts] == [333, 333, 334]
    m, C, x0, v0 = workloads.c1()
    assert (C / m == 1012.5).all()


def test_chain_launch_plan(lib):
    """osc_chain_plan needs no device: the C3/C4 plans the bench reports."""
    from paper_1702_02207_b200 import batched

    c3 = batched.chain_plan(1, 1 << 24, 10_000)
    # T = 31 fits 8720 tiles in 59 rounds of 148 CTAs (T = 32: 8739 tiles, 60)
    assert c3["steps_per_launch"] == 31 and c3["launches"] == 323
    assert c3["owned_per_tile"] == 2048 - 4 * 31 and c3["tiles_per_chain"] == 8720
    assert batched.chain_plan(1, 1 << 24, 10_000, halo_steps=32)["tiles_per_chain"] == 8739
    c4 = batched.chain_plan(4096, 1024, 10_000)
    assert (c4["cells_per_thread"], c4["threads"], c4["steps_per_launch"], c4["launches"]) == \
        (8, 128, 512, 20)
    with pytest.raises(ValueError):
        batched.chain_plan(1, 1 << 20, 100, halo_steps=600)


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of osc_peer_t / osc_edge_sync_t / osc_shard_t have
    the C layout (sizes and field offsets from a compiled probe)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:  # pragma: no cover
        pytest.skip("no C compiler")
    src = tmp_path / "probe.c"
    src.write_text('''
#include <stddef.h>
#include <stdio.h>
#include "osc_b200.h"
int main(void) {
    printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(osc_peer_t), sizeof(osc_edge_sync_t),
           sizeof(osc_shard_t), offsetof(osc_shard_t, nx), offsetof(osc_shard_t, n),
           offsetof(osc_shard_t, ghost), offsetof(osc_shard_t, first_bad),
           offsetof(osc_shard_t, sync), offsetof(osc_shard_t, div2));
    return 0;
}
''')
    exe = tmp_path / "probe"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(t) for t in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    S = _native.Shard
    want = [ctypes.sizeof(_native.Peer), ctypes.sizeof(_native.EdgeSync), ctypes.sizeof(S),
            S.nx.offset, S.n.offset, S.ghost.offset, S.first_bad.offset, S.sync.offset,
            S.div2.offset]
    assert got == want
