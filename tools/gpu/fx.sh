for mu in 100 1000; do for red in nccl ordered; do
echo "C5_1e8 mu=$mu $red: $(timeout 300 python bench.py --config C5_1e8 --mu-bp $mu --force-exchange --reduce $red --steps 50 --warmup 5 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 2 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})')"
done; done
