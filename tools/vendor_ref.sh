#!/bin/bash
# Vendor the UNMODIFIED reference into baseline/_ref (git-ignored, travels to the
# GPU box with the gpurun snapshot): the package through pip (the one offline
# install the brief allows) plus its own test suite, so the GPU tests can run the
# reference's assertions with the b200 lane installed (tests/test_ref_hosted.py).
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference}
TMP=$(mktemp -d)
cp -r "$SRC/pkg" "$TMP/pkg"          # the build writes egg-info next to the sources
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/semflow_tests"
rm -rf "$TMP"
echo "vendored $(python -c 'import sys; sys.path.insert(0, "'"$ROOT"'/baseline/_ref"); import semflow, os; print(os.path.dirname(semflow.__file__))')"
