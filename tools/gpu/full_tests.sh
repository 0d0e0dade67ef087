# the whole GPU suite (as the driver runs it) + smoke
export ARC_ORACLE_THREADS=$(nproc)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke rc=$?
timeout 3000 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/full_tests.log 2>&1; echo tests rc=$?
tail -25 gpurun_out/full_tests.log
