timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | grep -E "^FAILED|Error|error" | head -5
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines"
ARC_SKETCH_SHAPE=1 $CMD > gpurun_out/plain_v1.log 2>&1 && ARC_SKETCH_SHAPE=1 ncu --set full --clock-control none --import-source on -k regex:k_ef_sketch -s 10 -c 1 -o gpurun_out/prof_sketch_warp_v1 $CMD > gpurun_out/ncu_v1.log 2>&1
ls -la gpurun_out/prof_sketch_warp_v1.ncu-rep
