# round-2 evidence: default bench, launch list under ncu, one --set full capture of
# the sketch and select kernels (each after the same command exited 0 without ncu)
python bench.py > gpurun_out/r2_bench_default.jsonl 2> gpurun_out/r2_bench_default.err; echo bench rc=$?
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --no-extras"
$CMD > gpurun_out/r2_plain_prof.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launches.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/r2_plain_prof2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ef_sketch|k_select_gather" -s 20 -c 2 -o gpurun_out/r2_prof_round $CMD > gpurun_out/r2_ncu_full.log 2>&1; echo full rc=$?
