# ncu of the 32B QKV GEMM at 512 tokens under three plans (1-wave split, 2 splits, stream-K).
mkdir -p gpurun_out/r02
for plan in 2,1 1,2 2,-1; do
  tag=$(echo $plan | tr ',-' '_m')
  LP_TIME_GEMM_PLAN=$plan ncu --set full --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/r02/qkv512_$tag python scripts/prof_dominant.py 512 512 3 0 qwen2.5-32b > gpurun_out/r02/qkv512_$tag.log 2>&1
done
for plan in 1,5 1,-1; do
  tag=$(echo $plan | tr ',-' '_m')
  LP_TIME_GEMM_PLAN=$plan ncu --set full --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/r02/down512_$tag python scripts/prof_dominant.py 512 512 3 3 qwen2.5-32b > gpurun_out/r02/down512_$tag.log 2>&1
done
ls -la gpurun_out/r02/*512_*.ncu-rep
