#!/bin/bash
# Debug-build memory-safety pass, standing in for compute-sanitizer memcheck
# (not allowed on the GPU pool): rebuild with every gather index checked
# against its extent (er_idx in csrc/common.cuh), run the GPU suite and the
# all-kernel exercise, and require the device fault counters to stay at zero
# (tests/conftest.py checks after every GPU test).  GPU box only: it leaves
# the checked build in _lib/; rebuild without the flag afterwards.
set -e
export ER_NVCC_EXTRA="-DER_BOUNDS_CHECK=1"
python -c "from paper_2504_19930_b200 import _build; _build.build()"
export ER_ASSERT_NO_BOUNDS_FAULTS=1
python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@"
python tools/sanitize_target.py
unset ER_NVCC_EXTRA
python -c "from paper_2504_19930_b200 import _build; _build.build()"
