#!/bin/bash
# C2 probe + C5 (256^3) sweep points for each variant (run on the GPU box)
set -e
for v in "$@"; do
  ER_NVCC_EXTRA="$v" python paper_2504_19930_b200/_build.py > /dev/null
  echo "== $v"; python tools/measure_probe.py 2000 f32 3 2>&1 | tail -1
  python - <<'PY'
import sys, json
sys.argv = ["x"]
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import bench_configs
r = bench_configs.c5(pmax=16384)
print("C5", json.dumps([(x["particles"], round(x["evals_per_s"] / 1e9, 1)) for x in r["rows"]]))
PY
done
python paper_2504_19930_b200/_build.py > /dev/null
