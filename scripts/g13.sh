make -s -C oracle synth
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_forward_gpu.py -x -q 2>&1 | tail -3
for s in "256 1" "16 1" "128 8" "512 1"; do timeout 300 python scripts/prof_forward.py $s 0 qwen2.5-32b; done
