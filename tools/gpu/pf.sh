python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_select_modes.py -q -x 2>&1 | tail -1
LIBS="pf= nopf=ab/nopf/libarctopk.so" CONFIGS="C3 C2 C5_1e9" REPS=3 STEPS=200 bash tools/ab_probe.sh 2>&1
LIBS="pf= nopf=ab/nopf/libarctopk.so" CONFIGS="C4" REPS=2 STEPS=30 bash tools/ab_probe.sh 2>&1
timeout 300 python tools/stamps_probe.py C3 2>&1 | tail -8
