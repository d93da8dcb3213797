#!/bin/bash
# The one offline install of the reference (BASELINE / task contract): the
# unmodified tilefusion package into baseline/_ref (git-ignored, it travels
# to the GPU box with gpurun), plus a copy of its test suite into
# baseline/_ref_tests for tests/test_gpu_reference_shim.py.  Needs
# /root/reference (this container only).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/tilefusion_src && cp -r /root/reference/pkg /tmp/tilefusion_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/tilefusion_src
rm -rf baseline/_ref_tests && cp -r /root/reference/pkg/tests baseline/_ref_tests
echo "installed: $(ls baseline/_ref) + baseline/_ref_tests"
