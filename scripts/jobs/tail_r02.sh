mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_full_depth_gpu.py > gpurun_out/r02/tail_suite.log 2>&1; echo "rc=$?" >> gpurun_out/r02/tail_suite.log
bash scripts/jobs/attn_r02.sh tail
timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 8192 > gpurun_out/r02/tail_decompose.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_tail20.json 2> gpurun_out/r02/bench_tail20.err
