set -x
export ARC_ORACLE_THREADS=$(nproc)
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_ddp.py -x -q -k "loopback or ddp or ledger or placement" > gpurun_out/r2a_new.log 2>&1; echo new rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "graph" >> gpurun_out/r2a_new.log 2>&1; echo graph rc=$?
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/r2a_bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/r2a_new.log
