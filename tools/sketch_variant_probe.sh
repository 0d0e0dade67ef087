#!/bin/bash
# streaming-pass variant A/B (ARC_SKETCH_SHAPE 0/1/2, see arc_sketch.cu)
run() { timeout 600 python bench.py --steps ${STEPS:-200} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
for cfg in C3 "C2 --nodes-per-gpu 8 --pool 2" "C5_1e8 --pool 4" "C4 --steps 30 --pool 1"; do
  for sh in ${SHAPES:-0 1 2}; do
    echo "$cfg variant=$sh: $(ARC_SKETCH_SHAPE=$sh run --config $cfg)"
  done
done
