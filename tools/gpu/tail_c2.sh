python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tail.py -q -x 2>&1 | tail -2
for cfg in C5_1e6 C2; do for v in "ARC_TAIL=1" "ARC_TAIL=0"; do echo "$v: $(env $v timeout 300 python tools/graph_step_probe.py $cfg 2>&1 | tail -1)"; done; done
echo "base2 C5_1e6: $(ARC_LIB_PATH=ab/base2/libarctopk.so timeout 300 python tools/graph_step_probe.py C5_1e6 2>&1 | tail -1)"
timeout 300 python tools/tail_stamps.py C2 2>&1 | tail -3
