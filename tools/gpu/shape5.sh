python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
ENV_s5="ARC_SKETCH_SHAPE=5" ENV_s5nf="ARC_SKETCH_SHAPE=5" ENV_s2="ARC_SKETCH_SHAPE=2" LIBS="s0= s5= s5nf=ab/nofast/libarctopk.so s2=" CONFIGS="C3" REPS=3 STEPS=300 bash tools/ab_probe.sh 2>&1
ENV_s5="ARC_SKETCH_SHAPE=5" LIBS="def= s5=" CONFIGS="C5_1e9 C4" REPS=1 STEPS=30 bash tools/ab_probe.sh 2>&1
