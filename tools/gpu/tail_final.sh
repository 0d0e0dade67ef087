python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_select_modes.py tests/test_gpu_graph.py -q -x 2>&1 | tail -2
for v in "ARC_TAIL=1" "ARC_TAIL=0"; do echo "$v: $(env $v timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"; done
