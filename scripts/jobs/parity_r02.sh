# Full-depth parity tests + the whole GPU suite; numbers to gpurun_out/r02/.
mkdir -p gpurun_out/r02
export LP_PARITY_OUT=gpurun_out/r02/full_depth_parity.jsonl
rm -f $LP_PARITY_OUT
timeout 1500 python -m pytest tests/test_full_depth_gpu.py -x -q -s > gpurun_out/r02/full_depth.log 2>&1
echo "rc=$?" >> gpurun_out/r02/full_depth.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_full_depth_gpu.py > gpurun_out/r02/gpu_suite.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gpu_suite.log
bash scripts/jobs/decompose_r02.sh
