#!/usr/bin/env bash
# Install the UNMODIFIED reference package (oscbench) into baseline/_ref/, the
# one offline install this task allows.  baseline/_ref/ is git-ignored (not
# product source) but not gpurun-ignored, so it travels to the GPU box, where
# /root/reference does not exist.  The reference's own tests/ and configs/
# sit next to the installed package (tests/../configs is where
# test_acceptance.py:50,311 looks), so `tests/test_reference_suite.py` can run
# the reference's suite on the B200 with integrate/rk4_step rebound
# (paper_1702_02207_b200/dropin.py).
#
# The package needs only numpy, which the image has, hence --no-deps (pip's
# resolver cannot see the venv's numpy from --no-index).  The build writes
# into its source tree, so it installs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d /tmp/oscbench_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC/." "$TMP/"
rm -rf "$DST"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DST" "$TMP"
cp -r "$SRC/tests" "$DST/tests"
cp -r "$SRC/configs" "$DST/configs"
find "$DST" -name __pycache__ -prune -exec rm -rf {} +
echo "installed oscbench into $DST"
