python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/tail_stamps.py C5_1e6 > gpurun_out/tail_stamps.log 2>&1
for cfg in C5_1e6; do
  for tl in 1 0; do
  ARC_TAIL=$tl timeout 300 python bench.py --config $cfg --steps 200 --warmup 20 --no-baselines --no-extras --no-cpu-baseline --e2e-steps 2 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"][:8], "tail='$tl'", round(d["ms_per_step"]*1000,2), "us", d.get("p50_ms"), {k: round(v*1000,2) for k,v in d.get("phases_ms").items()})' >> gpurun_out/tail_bench2.log
  done
done
cat gpurun_out/tail_stamps.log gpurun_out/tail_bench2.log
