python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
ENV_s0="ARC_SKETCH_SHAPE=0" LIBS="def= s0=" CONFIGS="C3" ARGS="--force-exchange" REPS=2 STEPS=200 bash tools/ab_probe.sh 2>&1
ENV_s0="ARC_SKETCH_SHAPE=0" LIBS="def= s0=" CONFIGS="C3" ARGS="--force-exchange --reduce ordered" REPS=1 STEPS=200 bash tools/ab_probe.sh 2>&1
timeout 300 python tools/stamps_probe.py C3 2>&1 | tail -9
