python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
CMD="python bench.py --config C5_1e6 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-baselines --no-extras"
$CMD > gpurun_out/r02g_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ef_sketch|k_tail_update" -s 10 -c 2 -o gpurun_out/r02g_tail $CMD > gpurun_out/r02g_ncu.log 2>&1; echo ncu rc=$?
ls -la gpurun_out/r02g_tail.ncu-rep
