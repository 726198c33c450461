make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in "512 1" "256 4" "128 8"; do timeout 300 python scripts/prof_forward.py $s 0 qwen2.5-32b; done
for s in "512 1" "256 4" "128 8" "16 1"; do timeout 300 python scripts/prof_forward.py $s 0 qwen2.5-7b; done
