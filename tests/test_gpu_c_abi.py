"""The boundary is a plain C ABI: a C program links libosc_b200.so through
include/osc_b200.h alone (no Python, no torch) and runs the hot path."""

import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
from conftest import bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_c_program_uses_the_abi(tmp_path, golden):
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else shutil.which("gcc")
    exe = str(tmp_path / "c_abi_demo")
    libdir = os.path.join(ROOT, "paper_1702_02207_b200")
    cmd = [gcc, "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-o", exe, "-L", libdir,
           "-l:libosc_b200.so", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    dump = str(tmp_path / "dump.bin")
    out = subprocess.run([exe, dump], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("ok:")
    m, C, x0, v0, x, v = np.fromfile(dump, np.float64).reshape(6, 2, -1)
    _, _, xo, vo, fb = oracle.c_rk4_batch2(m, C, x0, v0, 1e-4, 2000, sample=False)
    assert not fb.any()
    assert bits(x) == bits(xo) and bits(v) == bits(vo)
    # the diverging canonical system (dt = 2e-2) is tagged at the reference's step
    step = int(out.stdout.split("tagged at step ")[1].split()[0])
    assert step == int(golden("edge")["div2e-2_first_bad"])
