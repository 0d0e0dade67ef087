#!/bin/bash
# A/B of the early gather (ARC_EARLY) and the slice size (ARC_SLICE_ROWS) on C3 / C2x8 / C5.
run() { timeout 600 python bench.py --steps ${STEPS:-200} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
for cfg in C3 "C2 --nodes-per-gpu 8 --pool 2" "C5_1e8 --mu-bp 1000 --pool 4" "C4 --steps 30 --pool 1"; do
  for e in 0 1; do
    for sr in "" 512 1024; do
      echo "$cfg early=$e slice=${sr:-auto}: $(ARC_EARLY=$e ARC_SLICE_ROWS=$sr run --config $cfg)"
    done
  done
done
