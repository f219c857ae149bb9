#!/bin/sh
# The one offline install of the reference the bench contract allows: the pure-Python bigmul
# package into baseline/_ref (git-ignored, shipped to the GPU box by gpurun), plus its test
# modules (baseline/_ref/reference_tests) so tests/test_reference_tests_on_device.py can run the
# reference's own DKSS tests against the device stages there.  /root/reference is read-only:
# install from a copy.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/bigmul_src "$ROOT/baseline/_ref"
cp -r /root/reference/pkg /tmp/bigmul_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" /tmp/bigmul_src
mkdir -p "$ROOT/baseline/_ref/reference_tests"
cp /tmp/bigmul_src/tests/*.py "$ROOT/baseline/_ref/reference_tests/"
rm -rf /tmp/bigmul_src
echo "installed bigmul into $ROOT/baseline/_ref"
