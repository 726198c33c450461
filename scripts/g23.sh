make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv --log-file gpurun_out/attn_long4.csv timeout 300 python scripts/attn_perf.py > /dev/null 2>&1
for t in 1 0; do LP_ATTN_TC=$t timeout 300 python scripts/prof_forward.py 256 16; LP_ATTN_TC=$t timeout 300 python scripts/prof_forward.py 16 1; done
