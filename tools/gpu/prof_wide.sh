# ncu --set full of the ranged (wide-row) sketch launch on P_n5461 (unaligned) and P_n5460 (aligned)
CMD="python bench.py --config P_n5461 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 1"
CMD2="python bench.py --config P_n5460 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 1"
$CMD > gpurun_out/plain_wide.log 2>&1 && $CMD2 >> gpurun_out/plain_wide.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ef_sketch -s 4 -c 1 -o gpurun_out/prof_n5461 $CMD > gpurun_out/ncu_wide.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ef_sketch -s 4 -c 1 -o gpurun_out/prof_n5460 $CMD2 >> gpurun_out/ncu_wide.log 2>&1
echo rc=$?
