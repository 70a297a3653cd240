"""Trajectory export.

* :func:`export_trajectory` -- the reference's CSV (harness.py:607-621): header
  ``t_s,x1_m,...,v1_mps,...``, ``%.9g`` fields, atomic temp+rename write
  (harness.py:548-558).  Byte-identical to ``oscbench.export_trajectory``.
* :func:`export_npz` -- lossless binary twin (times, positions, velocities):
  the CSV's 9 significant digits cannot round-trip a double.
* :func:`integrate_chains_to_npy` -- streaming export for runs whose samples
  do not fit in device memory: the integration proceeds one sampling
  interval at a time and each retained sample is copied device->pinned host
  on a side stream (overlapping the next interval's kernels) and written into
  a memory-mapped ``.npy`` of shape ``[nsamp][B][s]``.
"""

from __future__ import annotations

import os
import tempfile

import numpy as np


def _atomic_write(path: str, content: str):
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".oscb200-", suffix=".tmp")
    try:
        with os.fdopen(fd, "w", encoding="utf-8") as fh:
            fh.write(content)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def export_trajectory(traj, path: str):
    """CSV of a Trajectory, in the reference's exact format."""
    s = len(traj.samples[0].positions)
    if s == 2:
        header = "t_s,x1_m,x2_m,v1_mps,v2_mps"
    else:
        cols = [f"x{i + 1}_m" for i in range(s)] + [f"v{i + 1}_mps" for i in range(s)]
        header = "t_s," + ",".join(cols)
    lines = [header]
    for sample in traj.samples:
        row = [f"{sample.time:.9g}"]
        row += [f"{x:.9g}" for x in sample.positions]
        row += [f"{v:.9g}" for v in sample.velocities]
        lines.append(",".join(row))
    _atomic_write(path, "\n".join(lines) + "\n")


def export_npz(traj, path: str):
    """Lossless binary export: times [n], positions [n][s], velocities [n][s]."""
    times = np.array([smp.time for smp in traj.samples])
    xs = np.array([smp.positions for smp in traj.samples])
    vs = np.array([smp.velocities for smp in traj.samples])
    np.savez(path, times=times, positions=xs, velocities=vs, dt=traj.dt, stride=traj.stride)


def integrate_chains_to_npy(m, C, x0, v0, dt, nsteps, stride, path_prefix, *, halo_steps=0):
    """Integrate [B][s] chains, streaming every stride-th state to disk.

    Writes ``<prefix>.x.npy`` and ``<prefix>.v.npy`` ([1+nsteps//stride][B][s])
    and ``<prefix>.t.npy`` (accumulated time labels).  Returns the 1-based
    first bad step per chain (0: none); a diverged chain's samples after that
    step are unspecified, as integrate would have raised there.
    """
    import torch

    from . import batched
    from .oscillator import accumulated_times

    m, C, x, v = (batched._dev(a) for a in (m, C, x0, v0))
    if m.dim() == 1:
        m, C, x, v = (a[None] for a in (m, C, x, v))
    B, s = m.shape
    nsamp = 1 + nsteps // stride
    fx = np.lib.format.open_memmap(path_prefix + ".x.npy", mode="w+", dtype=np.float64,
                                   shape=(nsamp, B, s))
    fv = np.lib.format.open_memmap(path_prefix + ".v.npy", mode="w+", dtype=np.float64,
                                   shape=(nsamp, B, s))
    np.save(path_prefix + ".t.npy", accumulated_times(0.0, dt, nsteps, stride))
    copy_stream = torch.cuda.Stream()
    host = [(torch.empty((B, s), dtype=torch.float64).pin_memory(),
             torch.empty((B, s), dtype=torch.float64).pin_memory()) for _ in range(2)]
    done = [None, None]
    first_bad = torch.zeros(B, dtype=torch.int64, device=m.device)  # stays on the device

    def flush(slot, j):
        done[slot].synchronize()
        fx[j] = host[slot][0].numpy()
        fv[j] = host[slot][1].numpy()

    def enqueue(j, xs, vs):
        slot = j % 2
        if done[slot] is not None:
            flush(slot, j - 2)
        ev = torch.cuda.Event()
        ev.record()  # sample j is ready on the compute stream
        xs.record_stream(copy_stream)  # keep the caching allocator off it until copied
        vs.record_stream(copy_stream)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev)
            host[slot][0].copy_(xs, non_blocking=True)
            host[slot][1].copy_(vs, non_blocking=True)
            done[slot] = torch.cuda.Event()
            done[slot].record(copy_stream)
        return slot

    enqueue(0, x, v)
    k = 0
    j = 0
    while k < nsteps:
        n = min(stride, nsteps - k)
        res = batched.integrate_chains(m, C, x, v, dt, n, check=False, halo_steps=halo_steps,
                                       validate=(k == 0))
        fb = res.first_bad  # no host sync: the next interval queues behind this one
        first_bad = torch.where((first_bad == 0) & (fb > 0), fb + k, first_bad)
        x, v = res.x, res.v
        k += n
        if n == stride:
            j += 1
            enqueue(j, x, v)
    for jj in range(max(0, j - 1), j + 1):
        if done[jj % 2] is not None:
            flush(jj % 2, jj)
            done[jj % 2] = None
    fx.flush()
    fv.flush()
    return first_bad.cpu().numpy()
