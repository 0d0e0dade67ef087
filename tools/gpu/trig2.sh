python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
ENV_off="ARC_EARLY_TRIGGER=0" LIBS="on= off=" CONFIGS="C3 C2 C5_1e9 C5_1e8" REPS=3 STEPS=200 bash tools/ab_probe.sh 2>&1
ENV_off="ARC_EARLY_TRIGGER=0" LIBS="on= off=" CONFIGS="C4" REPS=2 STEPS=30 bash tools/ab_probe.sh 2>&1
