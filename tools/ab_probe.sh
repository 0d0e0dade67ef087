#!/bin/bash
# Interleaved A/B timing of library builds on the same box:
#   LIBS="old=ab/old/libarctopk.so new=" CONFIGS="C3 C5_1e8" bash tools/ab_probe.sh
# (an empty path = the in-tree build; extra env per label via ENV_<label>="K=V ...")
run() { timeout 600 python bench.py --steps ${STEPS:-150} --warmup 10 --e2e-steps 2 --no-cpu-baseline --no-baselines "$@" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), {k:round(v*1000,1) for k,v in d["phases_ms"].items() if v>0.003})'; }
for rep in $(seq ${REPS:-2}); do
  for cfg in ${CONFIGS:-C3}; do
    for lv in ${LIBS:-cur=}; do
      label=${lv%%=*}; path=${lv#*=}
      envv=$(eval echo \${ENV_$label})
      echo "$cfg [$label] rep$rep: $(env ARC_LIB_PATH=$path $envv bash -c "$(declare -f run); run --config $cfg ${ARGS}")"
    done
  done
done
