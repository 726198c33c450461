mkdir -p gpurun_out/r02
for spec in "16 1" "64 1" "256 1" "256 4"; do
for e in - norm qkv attn norm,qkv,attn; do
  if [ "$e" = "-" ]; then unset LP_DEBUG_EMPTY; else export LP_DEBUG_EMPTY=$e; fi
  timeout 300 python scripts/decompose_graph.py qwen2.5-32b $spec >> gpurun_out/r02/decompose_graph32.txt 2>&1
done
done
unset LP_DEBUG_EMPTY
LP_BENCH_SHARE_GPU=1 LP_BENCH_MODEL=qwen2.5-7b timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02/bench_share4.json 2> gpurun_out/r02/bench_share4.err
