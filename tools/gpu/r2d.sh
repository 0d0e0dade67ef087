export ARC_ORACLE_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or shapes or multi_block or llama or randomized or rows_of_at_most" > gpurun_out/r2d_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2d_tests.log
CMD="python bench.py --config P_n5461 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 1"
$CMD > gpurun_out/plain_wide.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ef_sketch -s 4 -c 1 -o gpurun_out/prof_n5461b $CMD > gpurun_out/ncu_wide.log 2>&1
echo rc=$?
