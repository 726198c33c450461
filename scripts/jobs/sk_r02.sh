# Stream-K GEMM: parity + A/B timing against the split-K plans.
mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/r02/sk_test.log 2>&1
echo "rc=$?" >> gpurun_out/r02/sk_test.log
tail -5 gpurun_out/r02/sk_test.log
timeout 900 python scripts/sk_sweep.py qwen2.5-32b > gpurun_out/r02/sk_sweep.txt 2>&1
timeout 600 python scripts/sk_sweep.py qwen2.5-7b >> gpurun_out/r02/sk_sweep.txt 2>&1
cat gpurun_out/r02/sk_sweep.txt
timeout 900 python -m pytest tests/test_forward_gpu.py -q -x > gpurun_out/r02/sk_fwd.log 2>&1
echo "rc=$?" >> gpurun_out/r02/sk_fwd.log
tail -5 gpurun_out/r02/sk_fwd.log
