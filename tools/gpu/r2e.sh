export ARC_ORACLE_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or shapes or multi_block or llama or randomized or rows_of_at_most" > gpurun_out/r2e_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/r2e_tests.log
bash tools/gpu/probe_layouts.sh
