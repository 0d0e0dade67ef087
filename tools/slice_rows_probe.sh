#!/bin/bash
# ms/step vs the select kernel's slice height (ARC_SLICE_ROWS) on the small configs
for cfg in "--config C2 --nodes-per-gpu 1" "--config C5_1e6" "--config C3" "--config C2 --nodes-per-gpu 8 --pool 2"; do
  for rows in default 128 256 512 1024; do
    if [ $rows = default ]; then unset ARC_SLICE_ROWS; else export ARC_SLICE_ROWS=$rows; fi
    out=$(timeout 300 python bench.py --steps 200 --warmup 10 --e2e-steps 1 --no-cpu-baseline --no-baselines $cfg 2>/dev/null | grep '^{')
    echo "$cfg rows=$rows $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2), "us", {k: round(v*1000,1) for k,v in d["phases_ms"].items()})')"
  done
done
