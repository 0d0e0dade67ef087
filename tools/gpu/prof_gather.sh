CMD="python bench.py --config C5_1e8 --mu-bp 1000 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 1"
ARC_EARLY=0 $CMD > gpurun_out/plain_gather.log 2>&1 && \
ARC_EARLY=0 ncu --set full --clock-control none --import-source on -k regex:k_select_gather -s 4 -c 1 -o gpurun_out/prof_gather $CMD > gpurun_out/ncu_gather.log 2>&1
echo rc=$?
