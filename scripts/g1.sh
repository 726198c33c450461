nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -30
