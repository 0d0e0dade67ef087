run() { timeout 600 python bench.py --steps 300 --warmup 20 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
echo "C3: $(run --config C3)"
echo "C3: $(run --config C3)"
echo "C5_1e9: $(run --config C5_1e9 --pool 1 --steps 40)"
