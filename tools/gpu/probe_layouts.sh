# per-layout sketch throughput (the unaligned-row question): one line per config
for c in P_n2048 P_n5460 P_n5461 C4; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 0 --pool 2 \
   | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['phases_ms'].items()}, 'sketch GB/s', round(d['roofline']['achieved']), round(d['roofline']['frac'],3))"
done
