# GEMM epilogue rework: parity (GEMM + forward tests) and the per-CTA timeline.
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_forward_gpu.py -q -x > gpurun_out/r02/epi_test.log 2>&1
echo "rc=$?" >> gpurun_out/r02/epi_test.log
tail -3 gpurun_out/r02/epi_test.log
bash scripts/jobs/gemm_prof_r02.sh > /dev/null 2>&1
cat gpurun_out/r02/gemm_prof32.txt gpurun_out/r02/gemm_prof7.txt
