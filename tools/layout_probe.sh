#!/bin/bash
# streaming pass on single-block layouts with LLaMA row lengths (aligned 2048, unaligned 5461)
run() { timeout 600 python bench.py --steps ${STEPS:-100} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
for cfg in P_n2048 P_n5461 C5_1e8; do
  for sh in ${SHAPES:-0}; do echo "$cfg variant=$sh: $(ARC_SKETCH_SHAPE=$sh run --config $cfg --pool 2)"; done
done
