make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for s in "16 1" "64 1" "128 1" "256 1"; do timeout 300 python scripts/prof_forward.py $s; done 2>&1 | grep shape
