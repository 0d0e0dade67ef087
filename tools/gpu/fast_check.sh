python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/fast_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/fast_tests.log
for cfg in C5_1e6 C2; do for lib in ab/base/libarctopk.so ""; do echo "$cfg lib=$lib $(ARC_LIB_PATH=$lib timeout 300 python tools/graph_step_probe.py $cfg 2>&1 | tail -1)"; done; done
LIBS="base=ab/base/libarctopk.so new=" CONFIGS="C3 C2 C5_1e8 C5_1e9" REPS=2 STEPS=200 bash tools/ab_probe.sh 2>&1
