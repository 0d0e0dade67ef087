python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
CMD="python tools/bucket_probe.py"
$CMD > gpurun_out/bk_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 2000 -c 600 --log-file gpurun_out/bk_launches.csv $CMD > gpurun_out/bk_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/bk_plain.log
