run() { timeout 600 python bench.py --steps ${STEPS:-100} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' ; }
{
run --config C2 --nodes-per-gpu 8 --pool 2
run --config C2 --nodes-per-gpu 1
run --config C3
run --config C5_1e8 --pool 4
} > gpurun_out/sweep2.jsonl
