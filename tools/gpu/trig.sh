python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
LIBS="cur= trig=ab/trig/libarctopk.so" CONFIGS="C3 C2 C5_1e9" REPS=3 STEPS=200 bash tools/ab_probe.sh 2>&1
LIBS="cur= trig=ab/trig/libarctopk.so" CONFIGS="C4" REPS=2 STEPS=30 bash tools/ab_probe.sh 2>&1
for lib in "" ab/trig/libarctopk.so; do echo "C5_1e6 [$lib] $(ARC_LIB_PATH=$lib timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"; done
