#!/usr/bin/env bash
# Stage the unmodified reference package and its tests into baseline/_ref
# (git-ignored, NOT gpurun-ignored: it travels to the GPU box, where
# tests/test_gpu_reference_suite.py runs the reference's own tests against
# the B200 backend through the pytest shim). Build container only: needs the
# read-only /root/reference. Never committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF=/root/reference/pkg
DST="$ROOT/baseline/_ref"
rm -rf "$DST" /tmp/fvv_refpkg
cp -r "$REF" /tmp/fvv_refpkg          # the build writes egg-info into its source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" /tmp/fvv_refpkg
cp -r "$REF/tests" "$DST/tests"
echo "staged fvv $(PYTHONPATH=$DST python -c 'import fvv; print(fvv.__version__)') into $DST"
