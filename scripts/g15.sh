make -s -C oracle synth
timeout 120 python -m pytest tests/test_replay_gpu.py -x -q 2>&1 | tail -3
echo "rc=$?"
nvidia-smi --query-gpu=utilization.gpu,memory.used --format=csv
