"""Build the in-tree CUDA library ``libosc_b200.so`` for sm_100a.

Each ``csrc/*.cu`` is compiled with nvcc in parallel and linked into one
shared object next to this file, so it travels with the repo snapshot to the
GPU box.  ``--fmad=false`` keeps every a*b+c of the reference unfused (the
kernels also spell each operation as an explicit ``__d*_rn`` intrinsic).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libosc_b200.so")
BUILD = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", "-I" + os.path.join(HERE, "..", "include")]


# Per-source ptxas options (measured on the B200, profiles/r02/README.md): K1's
# throughput loops (k_batch2_wide.cu) schedule best at register-usage level 2
# (C2 47.62 -> 47.29 ms); its one-system builds (C1 93.8 -> 101.5 ns/step) and
# the chain kernels (C3 536 -> 585 ms) lose with it, so it is not a global flag.
PER_SOURCE_FLAGS = {"k_batch2_wide.cu": ["-Xptxas", "--register-usage-level=2"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: str = OUT,
          build_dir: str = BUILD) -> str:
    """Compile every csrc/*.cu and link ``out``.  ``extra``: additional nvcc
    flags (used by scripts/build_variants.py for compiler-option sweeps)."""
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "osc_b200.h"))
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers):
            # a variant build that sets the same option itself replaces the per-source one
            per = PER_SOURCE_FLAGS.get(os.path.basename(src), [])
            if any(f.split("=")[0] in [e.split("=")[0] for e in extra] for f in per
                   if f.startswith("--")):
                per = []
            jobs.append([nvcc(), *NVCC_FLAGS, *per, *extra, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True,
                                                                   text=True), jobs)):
            if verbose or res.returncode:
                print(" ".join(cmd))
                print(res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"nvcc failed on {cmd[-3]}")
    if force or jobs or _newer(out, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", out, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
