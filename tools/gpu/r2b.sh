# persistent selection: parity + perf check
export ARC_ORACLE_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent or llama7b or graph or c1_config0 or shapes or adversarial or multi_block or binary64 or torch_stable" > gpurun_out/r2b_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r2b_tests.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-baselines --no-cpu-baseline --no-extras > gpurun_out/r2b_bench.log 2>&1; echo bench rc=$?
for c in C2 C5_1e6 C5_1e8; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-baselines --no-cpu-baseline --no-extras --e2e-steps 2 | cut -c1-400 >> gpurun_out/r2b_bench.log 2>&1; done
