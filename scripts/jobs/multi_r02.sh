mkdir -p gpurun_out/r02
export LP_PARITY_OUT=gpurun_out/r02/full_depth_parity2.jsonl
rm -f $LP_PARITY_OUT
timeout 1500 python -m pytest tests/test_full_depth_gpu.py -q > gpurun_out/r02/full_depth2.log 2>&1
echo "rc=$?" >> gpurun_out/r02/full_depth2.log
# N = 2 spatial instances sharing GPU 0 (functional check of the multi-GPU path on a 1-GPU box)
LP_BENCH_SHARE_GPU=1 LP_BENCH_MODEL=qwen2.5-7b timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02/bench_share2.json 2> gpurun_out/r02/bench_share2.err
LP_BENCH_SHARE_GPU=1 LP_BENCH_MODEL=qwen2.5-7b timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02/bench_share2_torchrun.json 2> gpurun_out/r02/bench_share2_torchrun.err
