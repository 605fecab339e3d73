#!/bin/bash
# C2 probe + C1 mask registration time for each build variant (GPU box)
set -e
for v in "$@"; do
  ER_NVCC_EXTRA="$v" python paper_2504_19930_b200/_build.py > /dev/null
  echo "== $v"; python tools/measure_probe.py 2000 f32 3 2>&1 | tail -1
  python tools/bench_configs.py c1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 ms', round(d['gpu_registration_ms'],3), round(d['gpu_registration_ms_median'],3))"
done
python paper_2504_19930_b200/_build.py > /dev/null
