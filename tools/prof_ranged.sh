# ncu --set full of the second (wide-V) sketch launch on the P_n5460 probe, and
# of the main launch on P_n2048 for comparison
for cfg in P_n5460 P_n2048; do
CMD="python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines"
$CMD > gpurun_out/plain_$cfg.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_ef_sketch -s 10 -c 1 -o gpurun_out/prof_$cfg $CMD > gpurun_out/ncu_$cfg.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
