"""The boundary is a plain C ABI: a C program links libosc_b200.so through
include/osc_b200.h alone (no Python, no torch) and runs the hot path."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_c_program_uses_the_abi(tmp_path):
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else shutil.which("gcc")
    exe = str(tmp_path / "c_abi_demo")
    libdir = os.path.join(ROOT, "paper_1702_02207_b200")
    cmd = [gcc, "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-o", exe, "-L", libdir,
           "-l:libosc_b200.so", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("ok:")
