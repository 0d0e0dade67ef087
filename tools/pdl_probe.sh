run() { timeout 600 python bench.py --steps 300 --warmup 20 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), round(d["step_roofline"]["frac"],3))'; }
for i in 1 2; do echo "PDL=1 C3: $(ARC_PDL=1 run --config C3)"; echo "PDL=0 C3: $(ARC_PDL=0 run --config C3)"; done
echo "PDL=1 C2x8: $(ARC_PDL=1 run --config C2 --nodes-per-gpu 8 --pool 2)"; echo "PDL=0 C2x8: $(ARC_PDL=0 run --config C2 --nodes-per-gpu 8 --pool 2)"
