#!/bin/bash
# Recipe: install the UNMODIFIED reference package (pipekrylov, pure Python +
# numba) into baseline/_ref so it travels to the GPU box with the snapshot
# (git-ignored, not gpurun-ignored), and copy its own test suite to
# baseline/_ref_tests.  Used by `bench.py --impl reference` (the stock
# numba CPU path) and tests/test_gpu_reference_suite.py (the reference's
# tests run against the B200 drivers).  /root/reference is read-only, so the
# build runs from a copy under /tmp.  numba/numpy come from the image.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${PK_REFERENCE_PKG:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 0; }
TMP=$(mktemp -d /tmp/pkref.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$ROOT/baseline/_ref" "$ROOT/baseline/_ref_tests"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP" > "$TMP/pip.log" 2>&1 || { tail -5 "$TMP/pip.log"; exit 1; }
mkdir -p "$ROOT/baseline/_ref_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref_tests/"
rm -rf "$TMP"
echo "reference installed in baseline/_ref, tests in baseline/_ref_tests"
