#!/bin/sh
# Install the unmodified reference package (respamd, /root/reference/pkg)
# into baseline/_ref -- git-ignored, but it travels to the GPU box with the
# gpurun snapshot -- together with its own container and integrator tests
# (baseline/_ref/respamd_tests), which tests/test_gpu_dropin.py runs with this
# package swapped in.  Nothing of it is committed; run it where
# /root/reference exists.
set -e
cd "$(dirname "$0")/.."
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref --upgrade /root/reference/pkg
rm -rf baseline/_ref/respamd_tests
mkdir -p baseline/_ref/respamd_tests
cp /root/reference/pkg/tests/conftest.py /root/reference/pkg/tests/test_containers.py \
   /root/reference/pkg/tests/test_integrators.py baseline/_ref/respamd_tests/
echo "reference installed in baseline/_ref"
