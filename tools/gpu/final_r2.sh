# final round-2 check: smoke + the whole GPU suite, the default bench line, and the ncu
# launch list of the fused-tail step (C5 d = 1e6)
bash tools/gpu/full_tests.sh
timeout 900 python bench.py > gpurun_out/r02e_bench_default.jsonl 2> gpurun_out/r02e_bench_default.err; echo bench rc=$?
CMD="python bench.py --config C5_1e6 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --no-extras"
$CMD > gpurun_out/r02e_plain_tail.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_tail_launches.csv $CMD > gpurun_out/r02e_ncu_tail.log 2>&1; echo ncu rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02e_bench_default.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['p50_ms'], d['roofline']['frac'], d.get('roofline_select'), d['step_roofline']['frac'], d['clocks'])
for k,v in d['extra_workloads'].items(): print(k, v.get('ms_per_step'), v.get('roofline_frac'), (v.get('graph') or {}).get('ms_per_step'))
PY
