#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (multispin, pure Python) into
# baseline/_ref (git-ignored; it travels to the GPU box with the gpurun
# snapshot) and copies its test suite next to it, for:
#   - bench.py --impl reference / cpu_baseline (the reference Engine timed on host cores),
#   - tests/test_gpu_reference_suite.py (the reference's own tests against this package's Engine),
#   - the reference CLI over the GPU engine (paper_2404_16990_b200.cli / backend).
# Needs /root/reference (this build container only).  The build writes into
# its source tree, so it installs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
echo "reference installed: $(ls "$ROOT/baseline/_ref")"
