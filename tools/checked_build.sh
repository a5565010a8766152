#!/bin/sh
# The checked library (device bounds checks, RB_CHECK in csrc/common.cuh)
# into build/librespa_checked.so; run the GPU tests against it with
#   RB_LIB_PATH=build/librespa_checked.so python -m pytest tests -m gpu -s -q | grep -c "RB_CHECK failed"
set -e
cd "$(dirname "$0")/.."
mkdir -p build
RB_NVCC_EXTRA="-DRB_CHECKED" python -c "
import sys; sys.path.insert(0, '.')
from paper_2507_11172_b200 import build as b
print(b.build(out='build/librespa_checked.so'))"
