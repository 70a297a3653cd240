"""Build compiler-option variants of libosc_b200.so for a sweep on the GPU box:
paper_1702_02207_b200/_variants/<tag>/libosc_b200.so, selected at run time with
OSC_LIB=<path> (see scripts/gpu_sweep_ptxas.sh).  Same sources, same
--fmad=false: every variant is held to the same byte-exact tests."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_02207_b200 import build  # noqa: E402

VARIANTS = {
    "rul0": ["-Xptxas", "--register-usage-level=0"],
    "rul1": ["-Xptxas", "--register-usage-level=1"],
    "rul2": ["-Xptxas", "--register-usage-level=2"],
    "rul3": ["-Xptxas", "--register-usage-level=3"],
    "rul4": ["-Xptxas", "--register-usage-level=4"],
    "rul6": ["-Xptxas", "--register-usage-level=6"],
    "rul7": ["-Xptxas", "--register-usage-level=7"],
    "rul8": ["-Xptxas", "--register-usage-level=8"],
    "rul10": ["-Xptxas", "--register-usage-level=10"],
    "O2": ["-Xptxas", "-O2"],
    "c128": ["-DOSC_B2_CHUNK=128"],
    "c256": ["-DOSC_B2_CHUNK=256"],
    "c512": ["-DOSC_B2_CHUNK=512"],
    "c1024": ["-DOSC_B2_CHUNK=1024"],
    "c4096": ["-DOSC_B2_CHUNK=4096"],
    "u1": ["-DOSC_B2_UNROLL=1"],
    "u2": ["-DOSC_B2_UNROLL=2"],
    "u3": ["-DOSC_B2_UNROLL=3"],
    "u8": ["-DOSC_B2_UNROLL=8"],
    "pb2": ["-DOSC_PERSIST_BUFS=2"],  # K3 double-buffered (round 1) vs 3 buffers
}

if __name__ == "__main__":
    base = os.path.join(build.HERE, "_variants")
    for tag, flags in VARIANTS.items():
        if len(sys.argv) > 1 and tag not in sys.argv[1:]:
            continue
        d = os.path.join(base, tag)
        out = build.build(force=True, extra=flags, out=os.path.join(d, "libosc_b200.so"),
                          build_dir=os.path.join(d, "obj"))
        print(tag, out)
