#!/bin/bash
# Round evidence: default bench (3 runs), launch list under ncu, one --set full
# capture of the sketch and select kernels (each after the same command ran clean).
set -x
for i in 1 2 3; do python bench.py > gpurun_out/bench_default_$i.jsonl 2> gpurun_out/bench_default_$i.err; done
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines"
$CMD > gpurun_out/plain_prof.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain_prof2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ef_sketch|k_select_gather" -s 20 -c 2 -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/prof_round.ncu-rep gpurun_out/launches.csv
