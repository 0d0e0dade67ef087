export ARC_ORACLE_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -k "exchange or loopback or bf16 or lsa or multi_block or randomized or noef or randk" > gpurun_out/r2h_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/r2h_tests.log
bash tools/gpu/fx.sh
