for c in C3 C4 P_n5460 C2 C5_1e6; do echo "== $c"; timeout 300 python tools/stamps_probe.py $c 2>&1 | tail -9; done
