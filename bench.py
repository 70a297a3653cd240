"""Benchmark of the RK4 hot path on B200 (driver contract: one JSON line).

Default workload = BASELINE.json configs[1] ("C2"): 2^20 independent 2-DOF
systems, fp64, dt=1e-4, 10^4 RK4 steps, seeded synthetic inputs.  One bench
"step" = one full pass of the hot path over that batch (2.1e10 DOF-steps).
Metric: DOF-steps/s (whole job, all ranks).  --config C1/C3/C4 times the other
single-GPU configurations the same way (DESIGN.md lists their lines).

Multi-GPU (torchrun, one rank per GPU, NCCL): the ranks split the ONE
workload (strong scaling) -- C2 systems, C4 chains and C5
trajectory columns in contiguous slices with no data-path collective, C3 as
a 1-D domain decomposition with a ghost exchange every T steps; device time
is the max over ranks.  At N > 1 the default line also carries `sharded_c3`:
C3 over the same N ranks through the fused peer exchange.

--impl reference times the reference algorithm on the host CPU (the
byte-identical C restatement in oracle/, all host threads) on a bounded sample
of the same workload and reports the same metric.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1702_02207_b200 import workloads  # noqa: E402

METRIC = "DOF-steps/s"
UNIT = "DOF-steps/s"
HBM_BYTES_PER_DOF_STEP = 48  # read x,v,m,C + write x,v, one step per round trip
FLOPS_PER_DOF_STEP = {"C1": 38, "C2": 38, "C3": 42, "C4": 42, "C5": 4 * 2 * 4096}
# DP-pipe instructions per DOF-step in the hot loops: counted at run time in
# the library's SASS (scripts/sass_stats.py; hot-loop kernel, DOFs advanced
# per loop iteration), these constants only if cuobjdump is unavailable.
DP_INST_PER_DOF_STEP = {"C1": 42, "C2": 42, "C3": 43, "C4": 43, "C5": None}


def _k1_unroll() -> int:
    """Steps per hot-loop iteration of K1's two-systems build: the default of
    OSC_B2_UNROLL in k_batch2.cu (the library bench.py runs is built from it)."""
    import re

    src = os.path.join(ROOT, "paper_1702_02207_b200", "csrc", "k_batch2.cu")
    try:
        with open(src) as f:
            return int(re.search(r"#define OSC_B2_UNROLL (\d+)", f.read()).group(1))
    except (OSError, AttributeError):
        return 2


# (kernel, DOF-steps per hot-loop iteration): K1's NS=2 build unrolls its step
# loop by OSC_B2_UNROLL (k_batch2.cu), so one iteration is that many steps x 2
# systems x 2 DOFs.
DP_LOOP_KERNEL = {"C1": ("batch2_rk4_kernelILi1ELb0ELb1ELi256E", 2),
                  "C2": ("batch2_rk4_kernelILi2ELb0ELb0ELi256E", 4 * _k1_unroll()),
                  # the two-operation build (kD2): both of its loops (tested or
                  # not, warp by warp) issue 344 DP instructions per step
                  "C3": ("chain_tiles_persistentILi8ELi256ELb0ELb1E", 8),
                  "C4": ("chain_rk4_kernelILi8ELb0ELb0ELi128ELb1E", 8)}


def dp_inst_per_dof_step(config: str, div2_frac=None):
    """(count, source) for the roofline_fp64 denominator.  K1 has two hot
    loops (three- and two-operation division); div2_frac = the fraction of
    systems running the two-operation one weights them."""
    if config not in DP_LOOP_KERNEL:
        return None, None
    try:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import sass_stats

        kern, dofs = DP_LOOP_KERNEL[config]
        from paper_1702_02207_b200 import _native

        loops = sass_stats.dp_loops(_native.LIB_PATH, kern)
        if loops and div2_frac is not None and len(loops) >= 2:
            n3, n2 = loops[0], loops[-1]
            n = div2_frac * n2 + (1 - div2_frac) * n3
            return n / dofs, (f"SASS of {kern}...: {n2} (two-operation division, "
                              f"{div2_frac:.4f} of systems) / {n3} (three-operation) DP instr "
                              f"per hot-loop iteration / {dofs} DOF-steps")
        if loops:
            return loops[0] / dofs, (f"SASS of {kern}...: {loops[0]} DP instr per hot-loop "
                                     f"iteration / {dofs} DOF-steps")
    except Exception:  # noqa: BLE001 -- cuobjdump missing: fall back to the counted constant
        pass
    return DP_INST_PER_DOF_STEP[config], "constant (counted with scripts/sass_stats.py --loop)"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, config: str):
    """dram bytes per launch from the committed ncu --set full summary, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel, {}).get(config)
    except (OSError, ValueError):
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = None

    def _nvml_start(self) -> bool:
        """Sample through NVML in this process (the library nvidia-smi itself
        uses): a query every 100 ms from a thread, no second process attached
        to the GPU -- the nvidia-smi loop's samples each cost the step they
        landed in ~1.5 ms (one step in five of a C2 run).  OSC_BENCH_SMI=1
        keeps the nvidia-smi loop."""
        if os.environ.get("OSC_BENCH_SMI") == "1":
            return False
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            index = self.index
            if vis:  # NVML counts physical devices
                ids = [v.strip() for v in vis.split(",") if v.strip()]
                if index < len(ids) and ids[index].isdigit():
                    index = int(ids[index])
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)  # fails early if unsupported
        except Exception:  # noqa: BLE001 -- no NVML binding: the nvidia-smi loop
            return False
        self.nvml = {"stop": threading.Event()}

        def loop():
            while not self.nvml["stop"].is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = ["Active" if mask & bits[n] else "Not Active" for n in self.NAMES]
                    self.lines.append(", ".join([str(sm), str(mx)] + flags))
                except Exception:  # noqa: BLE001
                    pass
                self.nvml["stop"].wait(0.1)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()
        t_end = time.time() + 1.0
        while not self.lines and time.time() < t_end:
            time.sleep(0.005)
        if not self.lines:  # NVML answers nothing here: the nvidia-smi loop instead
            self.nvml["stop"].set()
            self.thread.join(timeout=2)
            self.nvml = None
            return False
        return True

    def __enter__(self):
        if self._nvml_start():
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # let nvidia-smi finish its driver initialisation (first sample)
            # before the timed region, so that it cannot land inside a step
            t_end = time.time() + 2.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml:
            self.nvml["stop"].set()
            self.thread.join(timeout=2)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "NVML (pynvml), every 100 ms during the timed region" if self.nvml
                          else "nvidia-smi -lms 200 during the timed region"}


# --------------------------------------------------------------------------
# workloads: inputs resident in HBM + one "step" of the hot path
# --------------------------------------------------------------------------

def workload_desc(name: str, world: int = 1, transport: str = "nccl", T=None) -> dict:
    """The `config` description of a workload (shared by both bench arms)."""
    split = "one seeded draw split into G contiguous slices, one per rank (no collective)"
    if name == "C2":
        return {"workload": "C2: 2^20 independent 2-DOF systems (eq. 2), SoA [2][B]",
                "systems": workloads.C2_B, "systems_per_gpu": workloads.C2_B // world,
                "sharding": split}
    if name == "C4":
        return {"workload": "C4: 4096 chains x 1024 cells, [B][s]",
                "chains": workloads.C4_B, "chains_per_gpu": workloads.C4_B // world,
                "cells_per_chain": workloads.C4_S, "sharding": split}
    if name == "C3":
        return {"workload": "C3: one wall-anchored chain of 2^24 cells",
                "cells": workloads.C3_S, "halo_steps": T,
                "sharding": f"{world} contiguous shards, 2T-cell ghost zones "
                            f"refreshed every T steps ({transport})"}
    if name == "C5":
        return {"workload": "C5: dense SPD system s=4096, A = M^-1 K, 1024 trajectories",
                "s": workloads.C5_S, "trajectories": workloads.C5_N,
                "trajectories_per_gpu": workloads.C5_N // world,
                "sharding": "M, K built once on rank 0 and broadcast; trajectory columns "
                            "split G ways (no collective per step)",
                "gemm_per_launch": "4096 x 4096 x 2048 fp64 (DMMA), RK4 epilogue fused"}
    if name == "C1":
        return {"workload": "C1: paper 2-DOF system, C/m=1012.5, 10^6 steps (latency)"}
    raise SystemExit(f"unknown config {name}")


# implementation details of a workload description, kept out of `config` so
# that both bench arms report the identical workload configuration
IMPL_KEYS = ("halo_steps", "sharding", "gemm_per_launch")


def shared_config(name: str, world: int) -> dict:
    """The workload configuration both arms report (identical by construction):
    sizes, dt, steps per bench step, the whole job's DOF-steps and how the N
    GPUs split it."""
    p = workloads.PARAMS[name]
    desc = {k: v for k, v in workload_desc(name, world).items() if k not in IMPL_KEYS}
    total = {"C1": 2 * world, "C2": 2 * workloads.C2_B, "C3": workloads.C3_S,
             "C4": workloads.C4_B * workloads.C4_S,
             "C5": workloads.C5_S * workloads.C5_N}[name]
    return dict(desc, dt=p.dt, nsteps_per_step=p.nsteps, dof_steps_per_step=total * p.nsteps,
                parallelism={"C1": f"replicas{world}",
                             "C3": f"shards{world}"}.get(name, f"dp{world}"))


def c5_broadcast(rank, world, device):
    """workloads.c5() built once, on rank 0, and broadcast ("A
    built per GPU from the seed or broadcast once" -- the 4096^2 QR is the
    expensive part).  Host arrays on every rank."""
    if world == 1:
        return workloads.c5()
    import torch
    import torch.distributed as dist

    s, N = workloads.C5_S, workloads.C5_N
    shapes = ((s,), (s, s), (s, N), (s, N))
    host = workloads.c5() if rank == 0 else None
    out = []
    nccl = dist.get_backend() == "nccl"
    for i, shape in enumerate(shapes):
        t = (torch.from_numpy(host[i]) if rank == 0
             else torch.empty(shape, dtype=torch.float64))
        if nccl:
            t = t.to(device)
        dist.broadcast(t, src=0)
        out.append(t.cpu().numpy())
    return tuple(out)


class Workload:
    def __init__(self, name, rank, device, halo, world=1, transport="nccl"):
        import torch

        from paper_1702_02207_b200 import batched

        self.name, self.batched, self.torch = name, batched, torch
        p = workloads.PARAMS[name]
        self.dt, self.nsteps = p.dt, p.nsteps
        self.halo = halo
        self.world = world
        if name == "C2":
            # strong split: rank r integrates systems
            # [rB/G, (r+1)B/G) of the one seeded draw; no collective
            arrays = workloads.c2()
            self.total_dof = arrays[0].size
            sl = workloads.part(workloads.C2_B, rank, world)
            arrays = tuple(np.ascontiguousarray(a[:, sl]) for a in arrays)
            self.kernel, self.launches = "batch2_rk4_kernel", 1
            self.desc = workload_desc(name, world)
        elif name == "C4":
            arrays = workloads.c4()
            self.total_dof = arrays[0].size
            sl = workloads.part(workloads.C4_B, rank, world)
            arrays = tuple(np.ascontiguousarray(a[sl]) for a in arrays)
            self.kernel = "chain_rk4_kernel<8>"
            # whole-chain launches of 512 steps; batches of >= 1024 chains run
            # as two halves on two streams (capi.cu): two launches per 512 steps
            halves = 2 if arrays[0].shape[0] >= 1024 else 1
            self.launches = halves * -(-p.nsteps // 512)
            self.desc = workload_desc(name, world)
        elif name == "C3":
            arrays = workloads.c3()
            self.total_dof = arrays[0].size
            # T per shard: the plan for the (largest) shard's owned cells, the
            # same on every rank (neighbours must agree on the ghost width)
            plan = batched.chain_plan(1, -(-workloads.C3_S // world), p.nsteps, halo)
            T = plan["steps_per_launch"]
            self.kernel = "chain_tiles_persistent<8,256>"
            self.launches = plan["launches"]
            self.world = world
            self.desc = workload_desc(name, world, transport, T)
            self.shard = None
            if world > 1 and transport == "nccl":
                self.launches = 2 * self.launches  # interior + one edge launch per period
        elif name == "C5":
            # m, K built ONCE (rank 0: the QR of a 4096^2 draw) and broadcast;
            # rank r integrates trajectory columns [rN/G, (r+1)N/G)
            arrays = c5_broadcast(rank, world, device)  # m, K, X0, V0
            self.total_dof = arrays[2].size
            sl = workloads.part(workloads.C5_N, rank, world)
            arrays = arrays[:2] + tuple(np.ascontiguousarray(a[:, sl]) for a in arrays[2:])
            self.kernel = "dense_rk4_gemm"
            # 2 GEMMs per step, each as two halves of column tiles on two streams
            # when there are >= 16 column tiles of 32 (k_dense.cu); + rowscale,
            # pack, unpack in gpu_launches
            self.gemm_halves = 2 if 2 * (workloads.C5_N // world) // 32 >= 16 else 1
            self.launches = 2 * self.gemm_halves * p.nsteps
            self.desc = workload_desc(name, world)
        elif name == "C1":
            arrays = workloads.c1()
            arrays = tuple(a[:, None] for a in arrays)
            self.total_dof = 2 * world  # replicas
            self.kernel, self.launches = "batch2_rk4_kernel", 1
            self.desc = workload_desc(name)
        else:
            raise SystemExit(f"unknown config {name}")
        self.host = arrays
        self.dev = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrays)
        if name != "C5":  # the parameter rule once, at setup (not inside timed steps)
            batched.validate_parameters(self.dev[0], self.dev[1])
        self.dof = int(arrays[0].size) if name != "C5" else int(arrays[2].size)
        if name == "C3" and world > 1:
            from paper_1702_02207_b200 import sharded

            # strong scaling: each rank owns s/world cells plus 2T-cell ghosts
            self.shard = sharded.ShardedChain(*self.dev, self.dt, halo_steps=T, device=device,
                                              transport=transport)
            lo, hi = self.shard.L.own
            self.shard_x0 = self.shard.x.clone()
            self.shard_v0 = self.shard.v.clone()
            self.dof = hi - lo
        self.dof_steps = self.dof * self.nsteps
        self.total_dof_steps = self.total_dof * self.nsteps

    def step(self):
        m, C, x0, v0 = self.dev
        if self.name == "C5":
            A = self.batched.rowscale(C, m)  # (m, K): A = M^-1 K, once per run
            return self.batched.integrate_dense(A, x0, v0, self.dt, self.nsteps, check=False)
        if self.name in ("C2", "C1"):
            return self.batched.integrate_batch2(m, C, x0, v0, self.dt, self.nsteps, check=False,
                                                 validate=False)
        if self.name == "C3" and self.shard is not None:
            sh = self.shard  # reset the shard to the initial state, then integrate
            sh.x.copy_(self.shard_x0)
            sh.v.copy_(self.shard_v0)
            sh.first_bad.zero_()
            return sh.run(self.nsteps)
        if self.name == "C3":
            return self.batched.integrate_chains(m[None], C[None], x0[None], v0[None], self.dt,
                                                 self.nsteps, check=False, validate=False,
                                                 halo_steps=self.halo)
        return self.batched.integrate_chains(m, C, x0, v0, self.dt, self.nsteps, check=False,
                                             validate=False)

    def fma_step(self):
        m, C, x0, v0 = self.dev
        b = self.batched
        if self.name == "C2":
            return lambda: b.integrate_batch2(m, C, x0, v0, self.dt, self.nsteps, fma=True,
                                              check=False, validate=False)
        if self.name == "C3":
            return lambda: b.integrate_chains(m[None], C[None], x0[None], v0[None], self.dt,
                                              self.nsteps, fma=True, check=False,
                                              validate=False, halo_steps=self.halo)
        return lambda: b.integrate_chains(m, C, x0, v0, self.dt, self.nsteps, fma=True,
                                          check=False, validate=False)

    # ---- end to end through the host-pointer C ABI --------------------------------
    def e2e_sharded(self, steps, warmup):
        """Sharded C3: pinned host shard -> H2D -> integrate with halo exchange -> D2H."""
        torch = self.torch
        sh = self.shard
        hx = self.shard_x0.cpu().pin_memory()
        hv = self.shard_v0.cpu().pin_memory()
        hm = sh.m.cpu().pin_memory()
        hC = sh.C.cpu().pin_memory()
        lo, hi = sh.L.own
        ox = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
        ov = torch.empty_like(ox)
        times = []
        for i in range(warmup + steps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            sh.m.copy_(hm, non_blocking=True)
            sh.C.copy_(hC, non_blocking=True)
            sh.x.copy_(hx, non_blocking=True)
            sh.v.copy_(hv, non_blocking=True)
            sh.first_bad.zero_()
            sh.run(self.nsteps)
            x, v = sh.owned()
            ox.copy_(x, non_blocking=True)
            ov.copy_(v, non_blocking=True)
            torch.cuda.synchronize()
            if i >= warmup:
                times.append(time.perf_counter() - t)
        return sum(times), 4 * hx.numel() * 8, 2 * ox.numel() * 8 + 8

    def e2e_dense(self, steps, warmup):
        """C5 through the public API: pinned host m, K, X0, V0 -> H2D -> rowscale +
        integrate_dense -> D2H of X, V."""
        torch = self.torch
        pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in self.host]
        outs = [torch.empty_like(pinned[2]).pin_memory() for _ in range(2)]
        dev = self.dev[0].device
        times = []
        for i in range(warmup + steps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            m, K, X0, V0 = (a.to(dev, non_blocking=True) for a in pinned)
            res = self.batched.integrate_dense(self.batched.rowscale(K, m), X0, V0, self.dt,
                                               self.nsteps, check=False)
            outs[0].copy_(res.x, non_blocking=True)
            outs[1].copy_(res.v, non_blocking=True)
            torch.cuda.synchronize()
            if i >= warmup:
                times.append(time.perf_counter() - t)
        return sum(times), sum(a.numel() for a in pinned) * 8, 2 * outs[0].numel() * 8

    def e2e(self, steps, warmup):
        if self.name == "C5":
            return self.e2e_dense(steps, warmup)
        if getattr(self, "shard", None) is not None:
            return self.e2e_sharded(steps, warmup)
        from paper_1702_02207_b200 import _native

        torch = self.torch
        lib = _native.lib()
        pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in self.host]
        m, C, x0, v0 = pinned
        x = torch.empty_like(x0).pin_memory()
        v = torch.empty_like(v0).pin_memory()
        if self.name in ("C2", "C1"):
            B = x0.shape[1]
            fb = torch.empty(B, dtype=torch.int64).pin_memory()
            call = lambda: lib.osc_rk4_batch2_host(  # noqa: E731
                m.data_ptr(), C.data_ptr(), x.data_ptr(), v.data_ptr(), B, self.dt,
                self.nsteps, self.nsteps, None, None, fb.data_ptr())
        else:
            B, s = (1, x0.numel()) if self.name == "C3" else x0.shape
            fb = torch.empty(B, dtype=torch.int64).pin_memory()
            call = lambda: lib.osc_rk4_chains_host(  # noqa: E731
                m.data_ptr(), C.data_ptr(), x.data_ptr(), v.data_ptr(), B, s, self.dt,
                self.nsteps, self.nsteps, None, None, fb.data_ptr())
        h2d = sum(t.numel() * 8 for t in pinned)
        d2h = 2 * x0.numel() * 8 + fb.numel() * 8
        times = []
        for i in range(warmup + steps):
            x.copy_(x0)
            v.copy_(v0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            rc = call()  # synchronous: H2D, kernels, D2H, stream sync
            dt = time.perf_counter() - t
            if rc not in (_native.OSC_OK, _native.OSC_NONFINITE):
                raise RuntimeError(_native.last_error())
            if i >= warmup:
                times.append(dt)
        return sum(times), h2d, d2h


def python_reference_baseline(name, host, dt, nsteps, budget_s=8.0):
    """The reference's OWN CPU path, timed: ``oscbench.integrate`` (the
    unmodified package installed in baseline/_ref) under a
    multiprocessing.Pool of all host cores, each process integrating distinct
    systems / chains of this workload (BASELINE.md's plan).  A
    bounded sample (about budget_s of wall time), reported as completed
    DOF-steps per second.  C3 is one chain: the reference integrates it on
    one core (its thread engine is slower); C5 has no reference path."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "oscbench", "__init__.py")):
        return {"unavailable": "baseline/_ref missing (scripts/install_reference.sh)"}
    if name == "C5":
        return {"unavailable": "the reference has no dense path (SPEC.md:8,188)"}
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    m, C, x0, v0 = host
    if name in ("C1", "C2"):
        units = [(m[:, b], C[:, b], x0[:, b], v0[:, b]) for b in range(min(m.shape[1], 100_000))]
        dof, steps = 2, nsteps
    elif name == "C4":
        units = [(m[b], C[b], x0[b], v0[b]) for b in range(m.shape[0])]
        dof, steps = m.shape[1], nsteps
    else:  # C3: a 2^16-cell prefix of the chain, one core
        k = 1 << 16
        units = [(m[:k], C[:k], x0[:k], v0[:k])]
        dof, steps, cores = k, nsteps, 1
    # calibrate the per-step cost on one unit, then size the sample
    _ref_integrate((ref, units[0], dt, 2))  # imports
    t = time.perf_counter()
    _ref_integrate((ref, units[0], dt, 50))
    per_step = (time.perf_counter() - t) / 50
    steps = int(max(1, min(steps, budget_s / per_step / 2)))  # >= 2 units per core
    n_units = int(max(1, min(len(units), cores * budget_s / (per_step * steps))))
    cores = min(cores, n_units)
    jobs = [(ref, u, dt, steps) for u in units[:n_units]]
    ctx = mp.get_context("fork")
    t = time.perf_counter()
    if cores > 1:
        with ctx.Pool(cores) as pool:
            done = sum(pool.map(_ref_integrate, jobs, chunksize=1))
    else:
        done = sum(_ref_integrate(j) for j in jobs)
    el = time.perf_counter() - t
    what = {"C1": "systems", "C2": "systems", "C4": "chains", "C3": "chain prefix"}[name]
    return {"value": done * dof / el, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{n_units} {what} x {steps} of {nsteps} steps, {dof} DOF each; "
                      f"oscbench.integrate (baseline/_ref, unmodified) in a "
                      f"multiprocessing.Pool({cores})" if cores > 1 else
                      f"{n_units} {what} x {steps} of {nsteps} steps, {dof} DOF; "
                      f"oscbench.integrate on one core"}


def _ref_integrate(job):
    """One unit through the reference's own integrate; returns steps done."""
    ref, (m, C, x0, v0), dt, steps = job
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import oscbench

    oscbench.integrate(oscbench.build_chain(list(m), list(C)),
                       oscbench.PhaseState(tuple(x0), tuple(v0)), dt, steps, steps)
    return steps


def sharded_c3_record(rank, world, device, backend, local, steps=2, warmup=2):
    """C3 over the same N ranks through the fused peer exchange:
    one 2^24-cell chain in N contiguous shards, ghost zones refreshed by the
    tile kernels' own peer stores, edge tiles ordered on the device.  Device
    time per step is the max over ranks."""
    import torch
    import torch.distributed as dist

    wl3 = Workload("C3", rank, device, 0, world, transport="peer")
    for _ in range(warmup):
        wl3.step()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    host = []
    for a, b in ev:
        a.record()
        wl3.step()
        b.record()
        host.append(wl3.shard.host_s_per_period)
    torch.cuda.synchronize()
    dev_s = sum(a.elapsed_time(b) for a, b in ev) * 1e-3
    dev_s = allreduce_max(dev_s, device, backend)
    host_us = allreduce_max(max(h or 0.0 for h in host) * 1e6, device, backend)
    sh = wl3.shard
    T, g = sh.T, sh.L.g
    periods = -(-wl3.nsteps // T)
    per_gpu = wl3.total_dof_steps * steps / dev_s / world
    fp64 = fp64_peak(local)
    dp, _ = dp_inst_per_dof_step("C3")
    sides = 2 if 0 < rank < world - 1 else 1
    rec = {
        "value": wl3.total_dof_steps * steps / dev_s, "unit": UNIT, "n_gpus": world,
        "ms_per_step": dev_s * 1e3 / steps, "steps": steps, "warmup": warmup,
        "transport": "peer: boundary cells stored by the tile kernel straight into the "
                     "neighbours' next-input ghost zones (CUDA IPC / NVLink), edge tiles "
                     "ordered on the device (osc_edge_sync_t), one launch per period",
        "halo_steps": T, "ghost_cells": g, "periods_per_step": periods,
        "halo_bytes_per_period": {"per_neighbour": 2 * g * 8, "rank0": 2 * g * 8 * sides},
        "host_us_per_period_max": host_us,
        "roofline_fp64": {"bound": "fp64_pipe", "unit": "TFLOP/s",
                          "achieved": per_gpu * FLOPS_PER_DOF_STEP["C3"] / 1e12,
                          "peak": fp64 / 1e12,
                          "frac": per_gpu * FLOPS_PER_DOF_STEP["C3"] / fp64,
                          "issue_frac": per_gpu * dp / fp64 if dp else None},
    }
    sh.close()
    return rec


def guarded_sharded_c3(line, rank, world, device, backend, local):
    """Run sharded_c3_record on every rank under a watchdog.  `line`: rank 0's
    finished JSON line (None on the other ranks); the record, or the error,
    goes into line["sharded_c3"].  The multi-process peer exchange has only
    ever run time-sliced on one GPU (gpurun has one), so the bench must
    survive its failure on a real N-GPU box: an exception on one rank leaves
    the others waiting in a collective, and then the watchdog ends this
    process -- rank 0 prints the line it already has, with the reason, first
    (the reference guards its stage barrier the same way: abort + watchdog,
    parallel.py:205-255)."""
    limit = float(os.environ.get("OSC_SHARDED_C3_LIMIT", "240"))
    lock = threading.Lock()
    state = {"done": False}

    def bail():
        with lock:
            if state["done"]:
                return
            state["done"] = True
            if line is not None:
                line["sharded_c3"] = {"error": f"no result within {limit:.0f} s: a rank failed "
                                               "or stalled in the sharded C3 side record"}
                print(json.dumps(line), flush=True)
            sys.stderr.write(f"bench: rank {rank}: sharded C3 side record abandoned after "
                             f"{limit:.0f} s\n")
            sys.stderr.flush()
            os._exit(0)

    timer = threading.Timer(limit, bail)
    timer.daemon = True
    timer.start()
    failed = None
    try:
        if os.environ.get("OSC_BENCH_FAIL_RANK") == str(rank):  # test hooks
            raise RuntimeError("injected failure (OSC_BENCH_FAIL_RANK)")
        if os.environ.get("OSC_BENCH_STALL_RANK") == str(rank):
            time.sleep(1e6)  # a rank that never arrives: the watchdogs end the job
        rec = sharded_c3_record(rank, world, device, backend, local)
    except Exception as exc:  # noqa: BLE001
        failed = rec = {"error": f"{type(exc).__name__}: {exc}"[:500]}
    with lock:
        if state["done"]:  # the watchdog is printing / exiting
            time.sleep(3600)
        state["done"] = True
    timer.cancel()
    if line is not None:
        line["sharded_c3"] = rec
    if failed is not None:
        # the other ranks may be inside a collective this rank never joined:
        # do not enter another one (destroy_process_group) -- report and leave
        if line is not None:
            print(json.dumps(line), flush=True)
        sys.stderr.write(f"bench: rank {rank}: sharded C3 side record failed: "
                         f"{failed['error']}\n")
        sys.stderr.flush()
        os._exit(0)


def cublas_dgemm(device_index):
    """cuBLAS DGEMM (torch.matmul float64) on the C5 GEMM shape: the library bar."""
    import torch

    M, K, N = workloads.C5_S, workloads.C5_S, 2 * workloads.C5_N
    a = torch.randn(M, K, dtype=torch.float64, device=device_index)
    b = torch.randn(K, N, dtype=torch.float64, device=device_index)
    for _ in range(2):
        a @ b
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(10):
        a @ b
    end.record()
    torch.cuda.synchronize()
    return 10 * 2.0 * M * K * N / (start.elapsed_time(end) * 1e-3)


def fp64_peak(device_index, mode=0):
    """Measured FP64 rate: DFMA lane-instructions/s (mode 0) or DMMA flops/s (mode 2)."""
    import torch

    from paper_1702_02207_b200 import _native

    lib = _native.lib()
    sink = torch.empty(1024, dtype=torch.float64, device=device_index)
    ops = ctypes.c_int64(0)
    stream = torch.cuda.current_stream().cuda_stream
    best = 0.0
    for it in (2000, 20000, 20000):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        rc = lib.osc_bench_fp64(it, mode, sink.data_ptr(), ctypes.byref(ops), stream)
        end.record()
        torch.cuda.synchronize()
        if rc:
            raise RuntimeError(_native.last_error())
        best = max(best, ops.value / (start.elapsed_time(end) * 1e-3))
    return best


def cpu_baseline(wl: Workload, budget_s: float = 12.0):
    """Reference algorithm (oracle C restatement, byte-identical to oscbench) on
    the host cores, on a bounded sample of the same workload."""
    import oracle

    cores = len(os.sched_getaffinity(0))
    m, C, x0, v0 = wl.host
    if wl.name in ("C2", "C1"):
        B = m.shape[1]
        # calibrate: a small run, then size the sample for ~budget_s
        nb = min(B, max(cores * 256, 1024))
        cal_steps = min(wl.nsteps, 1000)
        t = time.perf_counter()
        oracle.c_rk4_batch2_final(m[:, :nb], C[:, :nb], x0[:, :nb], v0[:, :nb], wl.dt, cal_steps,
                                  nthreads=cores)
        rate = 2 * nb * cal_steps / max(time.perf_counter() - t, 1e-6)
        nb = int(min(B, max(nb, budget_s * rate / (2 * wl.nsteps))))
        t = time.perf_counter()
        oracle.c_rk4_batch2_final(m[:, :nb], C[:, :nb], x0[:, :nb], v0[:, :nb], wl.dt, wl.nsteps,
                                  nthreads=cores)
        el = time.perf_counter() - t
        done = 2 * nb * wl.nsteps
        sample = f"{nb} of {B} systems x {wl.nsteps} steps (full horizon)"
    elif wl.name == "C4":
        Bc, s = m.shape
        nb = max(cores, 8)
        steps = min(wl.nsteps, 1000)
        t = time.perf_counter()
        oracle.c_rk4_chains(m[:nb], C[:nb], x0[:nb], v0[:nb], wl.dt, steps, sample=False,
                            nthreads=cores)
        el = time.perf_counter() - t
        done = nb * s * steps
        sample = f"{nb} of {Bc} chains x {steps} of {wl.nsteps} steps"
    elif wl.name == "C5":
        # no reference implementation: the numpy restatement
        # (fp64 BLAS on all cores) -- "restatement, not reference"
        m, K, X0, V0 = wl.host
        A = K / m[:, None]
        steps = 2
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
        t = time.perf_counter()
        oracle.dense_rk4(A, X0, V0, wl.dt, steps)
        el = time.perf_counter() - t
        done = X0.size * steps
        sample = (f"{steps} of {wl.nsteps} steps of the full s=4096 x 1024 system, numpy/BLAS "
                  "restatement (the reference has no dense path)")
        return {"value": done / el, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": sample}
    else:  # C3: the whole chain, cells split across threads per phase
        s = m.size
        steps = 20
        t = time.perf_counter()
        oracle.c_rk4_chain_mt(m, C, x0, v0, wl.dt, steps, nthreads=cores)
        el = time.perf_counter() - t
        done = s * steps
        sample = f"full {s}-cell chain x {steps} of {wl.nsteps} steps"
    return {"value": done / el, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": sample + " (oracle/rk4_oracle.c, byte-identical to oscbench.integrate)"}


# --------------------------------------------------------------------------

def time_side(fn, warm=2, reps=3) -> float:
    """Seconds per call of a side measurement (CUDA events, current stream)."""
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3 / reps


def side_config_records(device, local, fp64, flush, steps=3, warmup=3):
    """C3, C4 and C5 beside the default C2 line: each workload built and timed
    as its own --config line is (CUDA events per step on the launching
    stream, L2 flushed between steps, W warm-up steps), reported as
    DOF-steps/s with its binding roofline fraction.  A failure is recorded,
    not fatal to the line."""
    import torch

    out = {}
    with ClockSampler(local) as clocks:
        for name in ("C4", "C3", "C5"):
            try:
                wl = Workload(name, 0, device, 0, 1, "peer")
                n = 2 if name == "C5" else steps
                for _ in range(warmup):
                    wl.step()
                torch.cuda.synchronize()
                ms = []
                for _ in range(n):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    wl.step()
                    b.record()
                    torch.cuda.synchronize()
                    ms.append(a.elapsed_time(b))
                t = sum(ms) * 1e-3 / n
                rec = {"value": wl.dof_steps / t, "unit": UNIT, "ms_per_step": t * 1e3,
                       "steps": n, "warmup": warmup, "kernel": wl.kernel,
                       "config": shared_config(name, 1)}
                if name == "C5":
                    flops = 2.0 * workloads.C5_S * workloads.C5_S * 2 * workloads.C5_N * 2 * wl.nsteps
                    dmma = fp64_peak(local, mode=2)
                    rec["roofline"] = {"bound": "tensor", "frac": flops / t / dmma,
                                       "achieved": flops / t / 1e12, "peak": dmma / 1e12,
                                       "unit": "TFLOP/s"}
                else:
                    fl = FLOPS_PER_DOF_STEP[name] * wl.dof_steps / t
                    rec["roofline"] = {"bound": "fp64_pipe", "frac": fl / fp64,
                                       "achieved": fl / 1e12, "peak": fp64 / 1e12,
                                       "unit": "TFLOP/s"}
                out[name] = rec
                del wl
                torch.cuda.empty_cache()
            except Exception as exc:  # noqa: BLE001
                out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    out["clocks"] = clocks.summary()
    return out


def allreduce_max(value: float, device, backend: str) -> float:
    """Max over ranks (device times are taken per rank; the job's is the max)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64,
                     device=device if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    wl_name = args.config
    import oracle  # noqa: F401  (the reference arm is the CPU restatement)

    class HostOnly:
        pass

    wl = HostOnly()
    wl.name = wl_name
    p = workloads.PARAMS[wl_name]
    wl.dt, wl.nsteps = p.dt, p.nsteps
    wl.host = {"C2": workloads.c2, "C4": workloads.c4, "C3": workloads.c3, "C5": workloads.c5,
               "C1": lambda: tuple(a[:, None] for a in workloads.c1())}[wl_name]()
    budget = args.ref_budget
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        last = cpu_baseline(wl, budget_s=budget)
        if i >= args.warmup:
            vals.append(last["value"])
    value = statistics.median(vals)
    cfg = shared_config(wl_name, world)
    dof = cfg.get("dof_steps_per_step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        # one whole workload at the sampled rate (each timed step is a bounded sample)
        "ms_per_step": dof / value * 1e3 if dof and value else None,
        "higher_is_better": True, "scaling": "weak" if wl_name == "C1" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy PCG64, workloads.py)",
        "config": cfg,
        "impl_notes": {"execution": f"{last['cores']} host threads (rank 0 only)",
                       "ms_per_step": "the whole workload extrapolated from the sampled rate",
                       "arithmetic": "IEEE fp64 CPU restatement, byte-identical to "
                                     "oscbench.integrate"},
        "cpu_baseline": dict(last, value=value),
        # the reference's own Python integrate on all cores, beside the C port
        "cpu_baseline_reference": python_reference_baseline(wl_name, wl.host, wl.dt, wl.nsteps,
                                                            budget_s=budget),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def relaunch(n: int) -> int:
    """`bench.py --gpus N` started without torchrun: run it as N ranks, one per
    GPU, exactly as the driver launches it."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--halo", type=int, default=0, help="C3 steps per tiled launch")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="C3 multi-GPU ghost exchange: peer-memory stores fused into the "
                         "tile kernel (default), or NCCL P2P (the library baseline)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sharded-c3", action="store_true",
                    help="at N > 1, skip the sharded C3 sub-record of the default line")
    ap.add_argument("--ref-budget", type=float, default=8.0)
    ap.add_argument("--no-side", action="store_true",
                    help="at N = 1, skip the C3/C4/C5 side records of the default C2 line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: at least 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup()
    # OSC_BENCH_BACKEND=gloo runs several ranks on fewer GPUs (rank -> GPU
    # local % count) to exercise the multi-rank path on a one-GPU box; the
    # kernels of different ranks never wait on one another.  Default: NCCL,
    # one rank per GPU.
    backend = os.environ.get("OSC_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    # C1 is one serial 2-DOF system: at N > 1 every rank runs a replica
    # (DESIGN.md "replicas only"); no collective on the data path.

    wl = Workload(args.config, rank, device, args.halo, world, args.transport)
    fp64 = fp64_peak(local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > L2 (126 MB)

    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:  # started (and settled) before the barrier
        barrier()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the step's events
            starts[i].record()
            wl.step()
            ends[i].record()
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_s = sum(step_ms) * 1e-3
    if world > 1:
        dev_s = allreduce_max(dev_s, device, backend)

    e2e = None
    if not args.no_e2e:
        e2e_s, h2d, d2h = wl.e2e(max(1, min(args.steps, 5)), 1)
        n_e2e = max(1, min(args.steps, 5))
        if world > 1:
            e2e_s = allreduce_max(e2e_s, device, backend)
        e2e = {"value": wl.total_dof_steps * n_e2e / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "timing": "wall clock around the synchronous host-pointer C-ABI call "
                         "(pinned host buffers; H2D + kernels + D2H inside)"}

    cpu = cpu_py = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # reported baselines: a failure there must not cost the GPU line
        try:
            cpu = cpu_baseline(wl)
        except Exception as exc:  # noqa: BLE001
            cpu = {"unavailable": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            cpu_py = python_reference_baseline(wl.name, wl.host, wl.dt, wl.nsteps)
        except Exception as exc:  # noqa: BLE001
            cpu_py = {"unavailable": f"{type(exc).__name__}: {exc}"[:300]}

    fma_line = None
    if wl.name in ("C2", "C3", "C4") and world == 1:
        # the opt-in OSC_FMA arithmetic on the same workload (not bit-identical;
        # tolerance in DESIGN.md), for context beside the exact headline
        fs = time_side(wl.fma_step())
        fma_line = {"value": wl.dof_steps / fs, "unit": UNIT, "ms_per_step": fs * 1e3,
                    "arithmetic": "OSC_FMA: contracted a*b+c, x/m as x*(1/m); rel. error "
                                  "<= 1e-12 vs the reference after 1e4 steps (measured 7e-15)"}

    validation_line = None
    if wl.name in ("C1", "C2") and world == 1:
        # On-device validation of every system against its analytic two-mode
        # solution (modal.compare fused into the K1 time loop).
        m, C, x0, v0 = wl.dev
        stride = workloads.PARAMS[wl.name].stride if wl.name == "C1" else 1000
        sol = wl.batched.analytic_batch2(m, C, x0, v0)
        run = lambda: wl.batched.integrate_batch2(  # noqa: E731
            m, C, x0, v0, wl.dt, wl.nsteps, stride, compare=True, analytic=sol, check=False,
            validate=False)
        vs = time_side(run)
        err = run().errors
        validation_line = {
            "value": wl.dof_steps / vs, "unit": UNIT, "ms_per_step": vs * 1e3,
            "samples_per_system": 1 + wl.nsteps // stride,
            "max_abs_error_max": float(err.max_abs_error.max()),
            "rmse_max": float(err.rmse.max()),
            "what": "modal.compare of every system vs its analytic solution, accumulated in "
                    "the time loop (no samples written)"}

    side = None
    if wl.name == "C2" and world == 1 and not args.no_side:
        # the other single-GPU configurations, timed the same way in the same
        # run (so the driver's record carries them; their own lines: --config)
        side = side_config_records(device, local, fp64, flush)

    engine_line = None
    if wl.name == "C1":
        # The paper's architecture on the GPU: one warp, lanes as equations,
        # __syncwarp as the stage barrier; per-step latency distribution.
        from paper_1702_02207_b200 import engine
        from paper_1702_02207_b200.oscillator import PhaseState, build_chain

        m, C, x0, v0 = workloads.c1()
        run = engine.run_equation_engine(build_chain(m, C), PhaseState(x0, v0), wl.dt, 100_000,
                                         100_000, warmup=1000)
        st = run.latency
        engine_line = {"steps": 100_000, "warmup": 1000, "p50_ns": st.p50 * 1e9,
                       "p90_ns": st.p90 * 1e9, "p99_ns": st.p99 * 1e9, "max_ns": st.max * 1e9,
                       "mean_ns": st.mean * 1e9, "stddev_ns": st.stddev * 1e9,
                       "timer": "%globaltimer around each step (lane 0)"}

    if getattr(wl, "shard", None) is not None:
        wl.shard.close()  # collective: every rank releases its peer mappings
    if world > 1:
        dist.barrier()
    want_sharded_c3 = world > 1 and args.config == "C2" and not args.no_sharded_c3
    if rank != 0:
        if want_sharded_c3:
            guarded_sharded_c3(None, rank, world, device, backend, local)
        if world > 1:
            dist.destroy_process_group()
        return 0

    # whole-job throughput: every rank's DOF-steps (the ranks partition the
    # one workload, C1 replicas aside) over the slowest rank's device time
    value = wl.total_dof_steps * args.steps / dev_s
    per_gpu = wl.dof_steps * args.steps / dev_s
    launch_s = dev_s / (args.steps * wl.launches)
    hbm_peak, hbm_src = peaks()
    alg_bytes = HBM_BYTES_PER_DOF_STEP * wl.dof_steps / wl.launches
    achieved = alg_bytes / launch_s / 1e9
    traffic = ncu_traffic(wl.kernel, wl.name)
    if wl.name == "C5":
        # GEMM launches dominate: 2 per RK4 step, each [s x s] x [s x 2N] run
        # as gemm_halves launches of column tiles
        gemm_flops = (2.0 * workloads.C5_S * workloads.C5_S * 2 * (workloads.C5_N // world)
                      / wl.gemm_halves)
        launch_s = dev_s / (args.steps * wl.launches)
        dmma = fp64_peak(local, mode=2)
        achieved_tf = gemm_flops / launch_s / 1e12
        roofline = {
            "bound": "tensor", "achieved": achieved_tf, "peak": dmma / 1e12, "unit": "TFLOP/s",
            "frac": achieved_tf * 1e12 / dmma, "traffic": traffic, "kernel": wl.kernel,
            "launches_per_step": wl.launches, "algorithmic_flops_per_launch": gemm_flops,
            "note": "FP64 tensor cores (DMMA.8x8x4). peak = measured DMMA issue "
                    "microbenchmark (MEASURED_PEAKS.json has no FP64); library bar = cuBLAS "
                    "DGEMM on the same shape, measured live",
            "cublas_dgemm_tflops": cublas_dgemm(local) / 1e12,
        }
    div2_frac = None
    if wl.name in ("C1", "C2") and os.environ.get("OSC_DIV2", "1")[:1] != "0":
        # systems whose two masses admit the two-operation division
        cls = wl.batched.div2_classify(wl.dev[0])
        div2_frac = float(((cls[0] != 0) & (cls[1] != 0)).double().mean())
    dp, dp_src = dp_inst_per_dof_step(wl.name, div2_frac)
    dp_inst_rate = per_gpu * dp if dp else None
    # SURVEY 8d's figure: 48 B per DOF-step (one step per HBM round trip);
    # above 1.0 because the kernels keep the state on-chip for many steps --
    # kept as a labelled secondary field, not the binding roofline
    roofline_hbm = {
        "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
        "frac": achieved / hbm_peak, "algorithmic_bytes_per_launch": alg_bytes,
        "note": f"SURVEY 8d definition (48 B/DOF-step, one step per HBM round trip); peak "
                f"{hbm_src}.  Not binding: state stays in registers / shared memory across "
                f"steps, so HBM moves ~{HBM_BYTES_PER_DOF_STEP} B per launch-sized block, "
                f"not per step (ncu dram bytes: `traffic` of the roofline)",
    }
    if wl.name != "C5":
        flops_launch = FLOPS_PER_DOF_STEP[wl.name] * wl.dof_steps / wl.launches
        achieved_tf = flops_launch / launch_s / 1e12
        roofline = {
            "bound": "fp64_pipe", "achieved": achieved_tf, "peak": fp64 / 1e12,
            "unit": "TFLOP/s", "frac": achieved_tf * 1e12 / fp64, "traffic": traffic,
            "kernel": wl.kernel, "launches_per_step": wl.launches,
            "algorithmic_flops_per_launch": flops_launch,
            "algorithmic_flops_per_dof_step": FLOPS_PER_DOF_STEP[wl.name],
            "peak_source": "measured live: osc_bench_fp64 mode 0, independent DFMA chains on "
                           "every SM (lane-instructions/s; the same pipe issues DADD/DMUL). "
                           "MEASURED_PEAKS.json has no FP64 entry; profiles/r01/fp64_peaks.json "
                           "has the DFMA/DADD/DMMA sweep",
            "peak_note": "1 flop per DP lane-instruction: the bit-exact path cannot contract "
                         "a*b+c into an FMA (each reference operation rounds separately), so "
                         "the FMA-doubled 2 flop/inst peak is not reachable by construction",
            "issue_frac": dp_inst_rate / fp64 if dp_inst_rate else None,
            "dp_inst_per_dof_step": dp, "dp_count_source": dp_src,
            "note": "C1 is one serial system (latency-bound, SURVEY 8d): no roofline claim"
                    if wl.name == "C1" else
                    "launch duration = device step time / launches_per_step" +
                    (" (includes the ~0.3 ms division classify + launch-order partition)"
                     if wl.name == "C2" else ""),
        }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak" if wl.name == "C1" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy PCG64, workloads.py; no dataset exists)",
        "config": shared_config(wl.name, world),
        "impl_notes": dict({k: v for k, v in wl.desc.items() if k in IMPL_KEYS},
                           dof_steps_per_gpu_step=wl.dof_steps,
                           l2="flushed between timed steps (256 MiB memset outside step "
                              "events); state is register-resident within a step",
                           arithmetic=("IEEE fp64; GEMM summation order differs from CPU BLAS "
                                       "(rel. 1e-10 vs the restatement)" if wl.name == "C5"
                                       else "IEEE fp64, byte-identical to oscbench.integrate")),
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "cpu_baseline": cpu,
        "cpu_baseline_reference": cpu_py,
        "e2e": e2e,
        # + C5: rowscale, pack, unpack; C1/C2: the division classifier and the
        # two kernels of the launch-order partition (cub::DevicePartition)
        # C3/C4: the two-operation division table pass
        "gpu_launches": (wl.launches + {"C1": 3, "C2": 3, "C5": 3, "C3": 1, "C4": 1}[wl.name])
                        * args.steps,
        "clocks": clocks.summary(),
        "step_ms": step_ms,
    }
    if side is not None:
        line["side_configs"] = side
    if world > 1 and backend != "nccl":
        line["note"] = f"{world} ranks over {backend} on {torch.cuda.device_count()} GPU(s): " \
                       "a multi-rank path check, not a scaling measurement"
    if engine_line:
        line["equation_engine"] = engine_line
    if fma_line:
        line["fma_mode"] = fma_line
    if validation_line:
        line["validation"] = validation_line
    if want_sharded_c3:
        # last, and with the line complete: a rank that fails or stalls in
        # this side record costs the sub-record, never the line
        guarded_sharded_c3(line, rank, world, device, backend, local)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
