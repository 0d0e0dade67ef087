run() { timeout 600 python bench.py --steps ${STEPS:-100} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
for f in 1 0; do echo "fused=$f C3: $(ARC_FUSED_GATHER=$f run --config C3)"; done
for f in 1 0; do echo "fused=$f C5_1e9 mu=10%: $(ARC_FUSED_GATHER=$f run --config C5_1e9 --mu-bp 1000 --pool 1 --steps 30)"; done
for f in 1 0; do echo "fused=$f C5_1e8 mu=10%: $(ARC_FUSED_GATHER=$f run --config C5_1e8 --mu-bp 1000 --pool 4)"; done
