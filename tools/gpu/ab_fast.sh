LIBS="base=ab/base/libarctopk.so fast1=ab/fast1/libarctopk.so fast2=ab/fast2/libarctopk.so" CONFIGS="C3" REPS=3 STEPS=300 bash tools/ab_probe.sh > gpurun_out/ab_fast.log 2>&1
LIBS="base=ab/base/libarctopk.so fast1=ab/fast1/libarctopk.so" CONFIGS="C5_1e8 C2" REPS=2 STEPS=200 bash tools/ab_probe.sh >> gpurun_out/ab_fast.log 2>&1
cat gpurun_out/ab_fast.log
