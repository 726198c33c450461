python scripts/fwd7b_perf.py 2>&1 | tail -20
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b.csv -s 3000 -c 300 python scripts/fwd7b_perf.py > /dev/null 2>&1
echo ncu rc=$?
