# Final multi-instance checks on one GPU: plain process and torchrun, 2 instances sharing GPU 0.
mkdir -p gpurun_out/r02
LP_BENCH_MODEL=qwen2.5-7b LP_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02/multi_final_plain.json 2> gpurun_out/r02/multi_final_plain.err; echo "plain rc=$?"
LP_BENCH_MODEL=qwen2.5-7b LP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02/multi_final_trun.json 2> gpurun_out/r02/multi_final_trun.err; echo "torchrun rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r02/multi_final_plain.json", "gpurun_out/r02/multi_final_trun.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("n_gpus"), d.get("value"), d.get("e2e", {}).get("value"), d.get("config", {}).get("parallelism"))
    except Exception as e:
        print(f, "ERR", e)
PY
