run() { timeout 600 python bench.py --steps 200 --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
echo "G=1 fused:            $(run --config C3)"
echo "exchange path (nccl): $(run --config C3 --force-exchange)"
echo "exchange path (ord):  $(run --config C3 --force-exchange --reduce ordered)"
