python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tail.py -q -x 2>&1 | tail -2
for i in 1 2; do echo "$(timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"; done
timeout 300 python tools/tail_stamps.py C5_1e6 2>&1 | tail -2
