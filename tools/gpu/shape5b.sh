python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
ENV_s5="ARC_SKETCH_SHAPE=5" LIBS="def= s5=" CONFIGS="C2 C5_1e8" REPS=2 STEPS=300 bash tools/ab_probe.sh 2>&1
ENV_s5="ARC_SKETCH_SHAPE=5" LIBS="def= s5=" CONFIGS="C2" ARGS="--nodes-per-gpu 8 --pool 2" REPS=2 STEPS=100 bash tools/ab_probe.sh 2>&1
for v in "" "ARC_SKETCH_SHAPE=5"; do echo "C2 graph [$v]: $(env $v timeout 300 python tools/graph_step_probe.py C2 2>&1 | tail -1)"; done
