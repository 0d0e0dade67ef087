set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_tail.py -x -q 2>&1 | tail -15 > gpurun_out/tail_tests.log
for cfg in C5_1e6 C3 C2; do
  timeout 300 python bench.py --config $cfg --steps 200 --warmup 20 --no-baselines --no-extras --no-cpu-baseline --e2e-steps 2 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], "tail", round(d["ms_per_step"]*1000,2), "us", d.get("p50_ms"), d.get("phases_ms"), d["roofline"]["frac"])' >> gpurun_out/tail_bench.log
  ARC_TAIL=0 timeout 300 python bench.py --config $cfg --steps 200 --warmup 20 --no-baselines --no-extras --no-cpu-baseline --e2e-steps 2 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], "notail", round(d["ms_per_step"]*1000,2), "us", d.get("p50_ms"), d.get("phases_ms"), d["roofline"]["frac"])' >> gpurun_out/tail_bench.log
done
cat gpurun_out/tail_tests.log gpurun_out/tail_bench.log
