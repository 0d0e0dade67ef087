#!/bin/bash
# ncu --set full of the streaming kernel for two library builds (same box)
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --config ${CFG:-C3}"
for lv in ${LIBS}; do
  label=${lv%%=*}; path=${lv#*=}
  ARC_LIB_PATH=$path $CMD > gpurun_out/plain_$label.log 2>&1 && ARC_LIB_PATH=$path ncu --set full --clock-control none --import-source on -k regex:k_ef_sketch -s 10 -c 1 -o gpurun_out/prof_$label $CMD > gpurun_out/ncu_$label.log 2>&1
  ls -la gpurun_out/prof_$label.ncu-rep
done
