make -s -C oracle synth
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
timeout 600 python -m pytest tests/test_forward_gpu.py -x -q 2>&1 | tail -3
timeout 300 python scripts/gemm_perf.py
for s in "256 1" "16 1" "128 8" "256 64" "512 1"; do timeout 300 python scripts/prof_forward.py $s; done
