make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scripts/attn_perf.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn --csv --log-file gpurun_out/attn_long2.csv python scripts/attn_perf.py > /dev/null 2>&1
for s in "16 1" "256 16"; do timeout 300 python scripts/prof_forward.py $s; done
