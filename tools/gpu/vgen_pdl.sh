python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_tail.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_ddp.py -q -x 2>&1 | tail -2
for i in 1 2; do echo "$(timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"; echo "$(timeout 300 python tools/graph_step_probe.py C2 2>&1 | tail -1)"; done
ENV_off="ARC_PDL=0" LIBS="on=" CONFIGS="C3" REPS=2 STEPS=200 bash tools/ab_probe.sh 2>&1
