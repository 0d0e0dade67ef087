python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for v in "" "ARC_SLICE_ROWS=1440 ARC_CLUSTER_TALL=1" "ARC_SLICE_ROWS=1440" "ARC_SLICE_ROWS=2880 ARC_CLUSTER_TALL=1"; do echo "C2 [$v]: $(env $v timeout 300 python tools/graph_step_probe.py C2 2>&1 | tail -1)"; done
ARC_SLICE_ROWS=1440 ARC_CLUSTER_TALL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs and C2" 2>&1 | tail -2
