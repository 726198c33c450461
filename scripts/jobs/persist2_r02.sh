mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_full_depth_gpu.py > gpurun_out/r02/persist2_suite.log 2>&1; echo "rc=$?" >> gpurun_out/r02/persist2_suite.log
bash scripts/jobs/attn_r02.sh persist2
LP_ATTN_PERSIST=0 bash scripts/jobs/attn_r02.sh nopersist2
python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_persist20.json 2> gpurun_out/r02/bench_persist20.err
python bench.py --steps 40 --warmup 5 > gpurun_out/r02/bench_persist40.json 2> gpurun_out/r02/bench_persist40.err
