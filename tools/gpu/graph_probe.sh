python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for cfg in C5_1e6 C2 C1 C3; do for tl in 1 0; do ARC_TAIL=$tl timeout 300 python tools/graph_step_probe.py $cfg 2>&1 | tail -1; done; done > gpurun_out/graph_probe.log
timeout 300 python -m pytest tests/test_gpu_tail.py -q -x 2>&1 | tail -2 >> gpurun_out/graph_probe.log
cat gpurun_out/graph_probe.log
