python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_tail.py tests/test_gpu_graph.py -q -x 2>&1 | tail -1
for i in 1 2; do for lib in "" ab/base/libarctopk.so; do echo "[$lib] $(ARC_LIB_PATH=$lib timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"; done; done
timeout 300 python tools/tail_stamps.py C5_1e6 2>&1 | tail -2
