bash tools/gpu/full_tests.sh
timeout 900 python bench.py > gpurun_out/r02f_bench_default.jsonl 2> gpurun_out/r02f_bench_default.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02f_bench_default.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['p50_ms'], d['roofline']['frac'], d['roofline_select']['frac'], d['step_roofline']['frac'], d['clocks'])
for k,v in d['extra_workloads'].items(): print(k, v.get('ms_per_step'), v.get('roofline_frac'), (v.get('graph') or {}).get('ms_per_step'))
PY
