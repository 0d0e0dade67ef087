export ARC_ORACLE_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "not full_size and not binary64 and not torch_stable" > gpurun_out/r2f_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r2f_tests.log
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C3 C5_1e8" REPS=1 STEPS=200 ARGS="--no-extras --pool 4" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C5_1e8 C5_1e9" REPS=1 STEPS=50 ARGS="--no-extras --pool 2 --mu-bp 1000" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C4 P_n5460" REPS=1 STEPS=50 ARGS="--no-extras --pool 2" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
