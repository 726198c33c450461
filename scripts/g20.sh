python scripts/attn_perf.py
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:attn --csv --log-file gpurun_out/attn_long.csv python scripts/attn_perf.py > /dev/null 2>&1
