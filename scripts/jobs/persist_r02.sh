mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_replay_gpu.py -x -q > gpurun_out/r02/persist_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02/persist_test.log
bash scripts/jobs/attn_r02.sh persist
timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 8192 > gpurun_out/r02/persist_decompose.txt 2>&1
LP_ATTN_PERSIST=0 timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 8192 >> gpurun_out/r02/persist_decompose.txt 2>&1
