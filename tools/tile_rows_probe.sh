run() { timeout 600 python bench.py --steps 200 --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' ; }
for R in 32 31 30 28 24; do echo "R=$R $(ARC_TILE_ROWS=$R run --config C3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))')"; done
echo "auto $(run --config C3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))')"
