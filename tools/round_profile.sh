#!/bin/bash
# Round evidence: default bench (3 runs), launch list under ncu, one --set full
# capture of the sketch and select kernels (each after the same command ran clean),
# and one of the TMA-fed sketch launch on C4 (its unaligned down projections).
#   TAG=r02b bash tools/round_profile.sh
set -x
TAG=${TAG:-round}
for i in 1 2 3; do python bench.py > gpurun_out/${TAG}_bench_default_$i.jsonl 2> gpurun_out/${TAG}_bench_default_$i.err; done
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --no-extras"
$CMD > gpurun_out/${TAG}_plain_prof.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
$CMD > gpurun_out/${TAG}_plain_prof2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ef_sketch|k_select_gather" -s 20 -c 2 -o gpurun_out/${TAG}_prof_round $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
C4="python bench.py --config C4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --no-extras"
$C4 > gpurun_out/${TAG}_plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ef_sketch_tma" -s 3 -c 1 -o gpurun_out/${TAG}_prof_c4_tma $C4 > gpurun_out/${TAG}_ncu_c4.log 2>&1
ls -la gpurun_out/${TAG}_*.ncu-rep gpurun_out/${TAG}_launches.csv
