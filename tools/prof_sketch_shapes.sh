set -e
for sh in 3 4; do ARC_SKETCH_SHAPE=$sh timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pt_shape$sh.log 2>&1 || echo "shape $sh FAILED"; grep -E "passed|failed" gpurun_out/pt_shape$sh.log | tail -1; done
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines"
for sh in 1 3; do
  ARC_SKETCH_SHAPE=$sh $CMD > gpurun_out/plain_$sh.log 2>&1 && ARC_SKETCH_SHAPE=$sh ncu --set full --clock-control none --import-source on -k regex:k_ef_sketch -s 10 -c 1 -o gpurun_out/prof_sketch_s$sh $CMD > gpurun_out/ncu_s$sh.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
