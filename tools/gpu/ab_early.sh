for c in C4 P_n5460 C3; do echo "== $c"; timeout 300 python tools/stamps_probe.py $c 2>&1 | tail -8; done
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C3 C2 C5_1e6 C5_1e8 P_n5460" REPS=2 STEPS=200 ARGS="--no-extras --pool 4" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C4 C5_1e9" REPS=1 STEPS=50 ARGS="--no-extras --pool 2" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
ENV_noearly="ARC_EARLY=0" LIBS="early= noearly=" CONFIGS="C5_1e8 C5_1e9" REPS=1 STEPS=50 ARGS="--no-extras --pool 2 --mu-bp 1000" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
