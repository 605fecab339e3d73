#!/bin/bash
# f64 (parity-exact) and f32 measurement throughput on C2 per build variant (GPU box)
set -e
for v in "$@"; do
  ER_NVCC_EXTRA="$v" python paper_2504_19930_b200/_build.py > /dev/null
  echo "== $v"; python tools/measure_probe.py 2000 f64,f32 3 2>&1 | tail -2
done
python paper_2504_19930_b200/_build.py > /dev/null
