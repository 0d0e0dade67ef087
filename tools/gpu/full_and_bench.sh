# the whole GPU suite + smoke, then the default bench line
bash tools/gpu/full_tests.sh
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_default.jsonl
