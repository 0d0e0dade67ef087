#!/bin/bash
# Bench lines for the BASELINE configs beyond the default (run on a GPU box).
set -u
out=${1:-gpurun_out/sweep}
mkdir -p $(dirname $out)
run() { timeout 600 python bench.py --steps ${STEPS:-100} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' ; }
{
run --config C1 --nodes-per-gpu 4 --pool 2
run --config C2 --nodes-per-gpu 8 --pool 2
run --config C2 --nodes-per-gpu 1
run --config C3
run --config C3 --force-exchange --reduce nccl
run --config C3 --force-exchange --reduce ordered
run --config C3 --force-exchange --reduce lsa
run --config C4 --pool 2
run --config C5_1e6
run --config C5_1e8 --mu-bp 10 --pool 4
run --config C5_1e8 --pool 4
run --config C5_1e8 --mu-bp 1000 --pool 4
run --config C5_1e9 --mu-bp 10 --pool 2
run --config C5_1e9 --pool 2
run --config C5_1e9 --mu-bp 1000 --pool 2
} > ${out}.jsonl
