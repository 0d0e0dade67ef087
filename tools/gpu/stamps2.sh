echo "== early"; timeout 300 python tools/stamps_probe.py C5_1e8 1000 2>&1 | tail -8
echo "== noearly"; ARC_EARLY=0 timeout 300 python tools/stamps_probe.py C5_1e8 1000 2>&1 | tail -8
