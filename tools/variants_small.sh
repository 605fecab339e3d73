#!/bin/bash
# C1 probe (64^3 mask, 500 particles) + C2 probe per build variant (GPU box)
set -e
for v in "$@"; do
  ER_NVCC_EXTRA="$v" python paper_2504_19930_b200/_build.py > /dev/null
  echo "== $v"; python tools/c1_probe.py 2>&1 | tail -1
  python tools/measure_probe.py 2000 f32 3 2>&1 | tail -1
done
python paper_2504_19930_b200/_build.py > /dev/null
