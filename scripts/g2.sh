set -x
make -s -C oracle synth
timeout 900 python -m pytest tests/test_forward_gpu.py -x -q 2>&1 | tail -30
