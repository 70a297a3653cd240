"""bench.py's guard around the sharded C3 side record (N > 1): a rank that
fails or stalls there costs the sub-record, never the C2 line -- rank 0 prints
the line it already has exactly once and every rank exits 0.  The guard is
host logic (a timer, a lock, os._exit), so it is driven here without a GPU by
replacing the record function."""

import json
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

DRIVER = textwrap.dedent("""
    import json, sys, time
    sys.path.insert(0, {root!r})
    import bench
    mode, rank = sys.argv[1], int(sys.argv[2])
    def record(*a, **k):
        if mode == "ok":
            return {{"value": 1.0}}
        if mode == "raise":
            raise RuntimeError("boom")
        time.sleep(1e6)
    bench.sharded_c3_record = record
    line = {{"metric": "DOF-steps/s", "value": 2.0}} if rank == 0 else None
    bench.guarded_sharded_c3(line, rank, 2, None, "gloo", 0)
    if line is not None:
        print(json.dumps(line), flush=True)
""")


def run(mode, rank, limit="1"):
    env = dict(os.environ, OSC_SHARDED_C3_LIMIT=limit)
    return subprocess.run([sys.executable, "-c", DRIVER.format(root=ROOT), mode, str(rank)],
                          capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)


@pytest.mark.parametrize("mode,key", [("ok", "value"), ("raise", "error"), ("stall", "error")])
def test_rank0_prints_exactly_one_line(mode, key):
    out = run(mode, 0)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] == 2.0 and key in d["sharded_c3"]
    if mode == "raise":
        assert "boom" in d["sharded_c3"]["error"]
    if mode == "stall":
        assert "no result within" in d["sharded_c3"]["error"]


@pytest.mark.parametrize("mode", ["ok", "raise", "stall"])
def test_other_ranks_exit_quietly(mode):
    out = run(mode, 1)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == ""
