mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_full_depth_gpu.py > gpurun_out/r02/plan_suite.log 2>&1
echo "rc=$?" >> gpurun_out/r02/plan_suite.log
for M in qwen2.5-32b qwen2.5-7b; do timeout 300 python scripts/decompose_chunk.py $M 0 4096 >> gpurun_out/r02/plan_decompose.txt 2>&1; done
LP_BENCH_OUT=gpurun_out/r02/bench_plan python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_plan20.json 2> gpurun_out/r02/bench_plan20.err
python bench.py --steps 40 --warmup 5 > gpurun_out/r02/bench_plan40.json 2> gpurun_out/r02/bench_plan40.err
