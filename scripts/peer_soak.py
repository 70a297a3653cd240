"""Soak of the fused peer transport across real processes (one GPU, time-
sliced contexts): many consecutive sharded runs, every one checked byte for
byte against the single-GPU integration and bounded in time.

    python scripts/peer_soak.py --groups 20 --runs 30 --out profiles/r02/peer_soak

Each group spawns `world` processes (alternating 2 and 3) that perform
`runs` consecutive runs; a run is a fresh ShardedChain (IPC setup of
buffers and edge counters), one `run` of random length on a random chain,
the gather, and the teardown.  Every run is bounded twice: the device-side
edge waits time out (OSC_PEER_TIMEOUT_MS, here 20 s -> PeerTimeoutError)
and the parent kills a group that exceeds its wall budget.  Writes one JSON
line per run and a summary.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def _port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, seed, runs, transport, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      OSC_PEER_TIMEOUT_MS=os.environ.get("OSC_PEER_TIMEOUT_MS", "20000"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1702_02207_b200 import batched, sharded

    rng = np.random.default_rng([seed, 7])  # same draws on every rank
    for i in range(runs):
        s = int(rng.integers(20_000, 150_000))
        T = int(rng.integers(4, 41))
        nsteps = int(rng.integers(1, 131))
        crng = np.random.default_rng([seed, i])
        m = crng.uniform(0.5, 2.0, s)
        C = crng.uniform(500.0, 2000.0, s)
        x0, v0 = crng.standard_normal(s), crng.standard_normal(s)
        t0 = time.monotonic()
        rec = {"world": world, "seed": seed, "run": i, "s": s, "T": T, "nsteps": nsteps}
        try:
            tr = transport if transport != "mixed" else ("peer", "nccl")[i % 2]
            rec["transport"] = tr
            sh = sharded.ShardedChain(m, C, x0, v0, 1e-3, halo_steps=T, transport=tr)
            fb = sh.run(nsteps)
            x, v = sh.gather()
            rec["trace"] = sh.trace[-4:]
            rec["host_us_per_period"] = (None if sh.host_s_per_period is None
                                         else round(sh.host_s_per_period * 1e6, 2))
            sh.close()
            rec["seconds"] = round(time.monotonic() - t0, 4)
            if rank == 0:
                ref = batched.integrate_chains(m, C, x0, v0, 1e-3, nsteps)
                same = (x.numpy().tobytes() == ref.x[0].cpu().numpy().tobytes()
                        and v.numpy().tobytes() == ref.v[0].cpu().numpy().tobytes())
                rec["ok"] = bool(same and fb == 0)
        except Exception as exc:  # noqa: BLE001 - recorded, then the group stops
            rec["error"] = f"{type(exc).__name__}: {exc}"
            rec["ok"] = False
            if rank == 0:
                q.put(rec)
            raise
        if rank == 0:
            q.put(rec)
    dist.destroy_process_group()
    if rank == 0:
        q.put(None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=20)
    ap.add_argument("--runs", type=int, default=30)
    ap.add_argument("--budget", type=float, default=600.0, help="wall seconds per group")
    ap.add_argument("--out", default="gpurun_out/peer_soak")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl", "mixed"],
                    help="nccl: the NCCL-transport schedule (over gloo here); mixed: alternate")
    args = ap.parse_args()

    import queue as queue_mod

    import torch.multiprocessing as mp

    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    lines = open(args.out + ".jsonl", "w")
    ctx = mp.get_context("spawn")
    total = ok = bad = hung = 0
    worst = 0.0
    host_us = []
    t_start = time.monotonic()
    for gidx in range(args.groups):
        world = 2 + gidx % 2
        q = ctx.Queue()
        procs = mp.start_processes(_worker, args=(world, _port(), 1000 + gidx, args.runs,
                                                  args.transport, q),
                                   nprocs=world, join=False, start_method="spawn")
        deadline = time.monotonic() + args.budget
        done = False
        while not done:
            try:
                rec = q.get(timeout=1.0)
            except queue_mod.Empty:
                if time.monotonic() > deadline:
                    hung += 1
                    lines.write(json.dumps({"world": world, "seed": 1000 + gidx,
                                            "hang": True}) + "\n")
                    for p in procs.processes:
                        p.kill()
                    break
                try:
                    if procs.join(timeout=0):
                        break
                except Exception as exc:  # a rank died
                    lines.write(json.dumps({"world": world, "seed": 1000 + gidx,
                                            "died": str(exc)[:300]}) + "\n")
                    bad += 1
                    break
                continue
            if rec is None:
                done = True
                continue
            total += 1
            ok += bool(rec.get("ok"))
            bad += not rec.get("ok")
            worst = max(worst, rec.get("seconds", 0.0))
            if rec.get("host_us_per_period") is not None:
                host_us.append(rec["host_us_per_period"])
            lines.write(json.dumps(rec) + "\n")
            lines.flush()
        try:
            while not procs.join(timeout=30):
                pass
        except Exception:  # noqa: BLE001
            pass
    lines.close()
    summary = (f"{args.transport} transport soak: {total} runs ({args.groups} process groups of 2/3 ranks, "
               f"{args.runs} runs each) -> {ok} byte-exact, {bad} failed, {hung} hung groups; "
               f"slowest run {worst:.2f} s; host time per period (native loop) median "
               f"{(sorted(host_us)[len(host_us) // 2] if host_us else float('nan')):.1f} us; "
               f"wall {time.monotonic() - t_start:.0f} s")
    print(summary)
    with open(args.out + ".txt", "w") as f:
        f.write(summary + "\n")
    return 0 if (bad == 0 and hung == 0 and total == args.groups * args.runs) else 1


if __name__ == "__main__":
    raise SystemExit(main())
