LIBS="cur= ld0=ab/ld0/libarctopk.so ld4=ab/ld4/libarctopk.so" CONFIGS="C3 C5_1e8 C2 P_n5460 P_n5461" REPS=2 STEPS=200 ARGS="--no-extras --pool 4" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
LIBS="cur= ld0=ab/ld0/libarctopk.so" CONFIGS="C4" REPS=2 STEPS=50 ARGS="--no-extras --pool 2" bash tools/ab_probe.sh 2>&1 | grep -v Traceback
