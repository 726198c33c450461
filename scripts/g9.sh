timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
for mode in 0 2; do python scripts/gemm_one.py 37888 2048 3584 $mode 256 2 1 10; done
python scripts/gemm_one.py 37888 256 3584 2 256 2 1 10
python scripts/gemm_one.py 37888 128 3584 2 128 2 1 10
python scripts/gemm_one.py 37888 64 3584 2 64 1 1 10
python scripts/gemm_one.py 37888 16 3584 2 16 1 1 10
