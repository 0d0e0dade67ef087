python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for cfg in C5_1e6; do for v in "ARC_TAIL=1" "ARC_TAIL=1 ARC_TAIL_SHAPE=0" "ARC_TAIL=0"; do echo "$v: $(env $v timeout 300 python tools/graph_step_probe.py $cfg 2>&1 | tail -1)"; done; done > gpurun_out/graph_probe2.log
timeout 300 python tools/tail_stamps.py C5_1e6 >> gpurun_out/graph_probe2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tail.py tests/test_gpu_select_modes.py -q -x 2>&1 | tail -2 >> gpurun_out/graph_probe2.log
cat gpurun_out/graph_probe2.log
