make -s -C oracle synth
timeout 600 python -m pytest tests/test_forward_gpu.py -q -x 2>&1 | tail -15
timeout 300 python scripts/attn_perf.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv --log-file gpurun_out/attn_long3.csv timeout 300 python scripts/attn_perf.py > /dev/null 2>&1
