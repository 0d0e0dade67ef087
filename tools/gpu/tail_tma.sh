python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_tail.py -q -x 2>&1 | tail -3
for tl in 1 0; do ARC_TAIL=$tl timeout 900 python tools/bucket_probe.py 2>&1 | tail -1; ARC_TAIL=$tl timeout 900 python tools/bucket_probe.py graphs 2>&1 | tail -1; done
