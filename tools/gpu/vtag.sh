python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_tail.py tests/test_gpu_graph.py tests/test_gpu_ddp.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x 2>&1 | tail -2
for i in 1 2; do for c in C5_1e6 C2; do echo "$(timeout 300 python tools/graph_step_probe.py $c 2>&1 | tail -1)"; done; done
for g in "" graphs; do ARC_TAIL=1 timeout 900 python tools/bucket_probe.py $g 2>&1 | tail -1; done
