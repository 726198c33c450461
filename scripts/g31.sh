make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
K='regex:qkv_post'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 30 -c 10 --csv --log-file gpurun_out/qkvpost.csv python scripts/prof_forward.py 256 16 > /dev/null 2>&1
python scripts/summarize_ncu.py gpurun_out/qkvpost.csv | head -3
for s in "256 16" "16 1"; do timeout 300 python scripts/prof_forward.py $s; done 2>&1 | grep shape

ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 30 -c 10 --csv --log-file gpurun_out/qkvpost16.csv python scripts/prof_forward.py 16 1 > /dev/null 2>&1
python scripts/summarize_ncu.py gpurun_out/qkvpost16.csv | head -3
