#!/usr/bin/env bash
# Install the unmodified reference (flexep 0.1.0) into baseline/_ref (git-ignored; it travels
# to the GPU box with gpurun) and keep a copy of its own test files next to it, so the
# drop-in can be run against the reference's tests where /root/reference does not exist.
# Build container only (reads /root/reference, read-only: installed from a copy in /tmp).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
rm -rf /tmp/flexep_src && cp -r /root/reference/pkg /tmp/flexep_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade /tmp/flexep_src
rm -rf "$ROOT/baseline/_ref/reference_tests"
cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/reference_tests"
echo "flexep installed in $ROOT/baseline/_ref (tests in baseline/_ref/reference_tests)"
