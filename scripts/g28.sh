make -s -C oracle synth
echo "=== reference arm"
( time timeout 600 python bench.py --impl reference --steps 10 --warmup 3 ) 2>&1 | tail -4
echo "=== 2 ranks sharing GPU 0 (functional check)"
LP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 2>&1 | grep -v "^ \|Exception ignored\|Traceback\|ModuleNotFound\|W1017\|warnings.warn" | tail -3 | cut -c1-600
echo "=== reference arm under torchrun (rank 0 prints, others exit)"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 2>&1 | tail -2 | cut -c1-300
