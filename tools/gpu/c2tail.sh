python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for tl in 1 0; do echo "C2 ARC_TAIL=$tl $(ARC_TAIL=$tl timeout 300 python tools/graph_step_probe.py C2 2>&1 | tail -1)"; done
timeout 300 python tools/tail_stamps.py C2 2>&1 | tail -2
