"""SASS-level guards on the built library (CPU; needs cuobjdump, no GPU):
the hot loops keep the instruction counts DESIGN.md quotes, so a change that
silently re-inflates the arithmetic (an FMA contraction lost, the division
back to three operations) fails here before any GPU run."""

import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1702_02207_b200", "libosc_b200.so")

pytestmark = pytest.mark.skipif(not (shutil.which("cuobjdump") and os.path.exists(LIB)),
                                reason="needs cuobjdump and the built library")
sys.path.insert(0, os.path.join(ROOT, "scripts"))


@pytest.fixture(scope="module")
def kernels():
    """{mangled name: [(address, instruction)]}, one cuobjdump pass."""
    import sass_stats

    return dict(sass_stats.functions(LIB))


def _body(kernels, substr):
    return next(b for n, b in kernels.items() if substr in n)


def test_batch2_hot_loops(kernels):
    import sass_stats

    # K1's throughput build: the three-operation loop (84 DP per system-step)
    # and the two-operation loop (76), OSC_B2_UNROLL steps x 2 systems per
    # iteration -- the bit-exact minimum of 38 DP instructions per DOF-step
    import bench

    per_iter = 2 * (bench.DP_LOOP_KERNEL["C2"][1] // 4)   # system-steps per iteration
    loops = sass_stats.hot_loops(_body(kernels, "batch2_rk4_kernelILi2ELb0ELb0ELi256E"))
    assert loops[:2] == [84 * per_iter, 76 * per_iter], loops


def test_chain_hot_loops(kernels):
    import sass_stats

    for kern in ("chain_tiles_persistentILi8ELi256ELb0E", "chain_rk4_kernelILi8ELb0ELb0ELi128E",
                 "chain_rk4_kernelILi8ELb0ELb0ELi256E"):
        assert sass_stats.hot_loops(_body(kernels, kern))[0] == 47 * 8, kern


def test_no_local_memory_in_hot_loops(kernels):
    import re

    import sass_stats

    # every build of the time-step kernels (all shapes, FMA and compare
    # variants): a launch bound that caps registers too low shows up here
    for name, body in kernels.items():
        if not any(k in name for k in ("batch2_rk4_kernel", "chain_tiles_persistent",
                                       "chain_rk4_kernel")):
            continue
        for addr, ins in body:
            m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)\s*$", ins)
            if m and int(m.group(1), 16) < addr:
                seg = [i for a, i in body if int(m.group(1), 16) <= a <= addr]
                ops = {sass_stats.opcode(i) for i in seg}
                dp = sum(sass_stats.opcode(i) in ("DADD", "DMUL", "DFMA") for i in seg)
                if dp >= 40 and "CALL" not in ops:
                    assert not ops & {"LDL", "STL"}, name
