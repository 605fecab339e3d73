#!/bin/bash
# ziggurat table placement: C1 probe (predict every iteration) + device phantom timing
set -e
for v in "$@"; do
  ER_NVCC_EXTRA="$v" python paper_2504_19930_b200/_build.py > /dev/null
  echo "== $v"; python tools/c1_probe.py 2>&1 | tail -1
  python tools/phantom_timing.py 2>&1 | tail -3
done
python paper_2504_19930_b200/_build.py > /dev/null
