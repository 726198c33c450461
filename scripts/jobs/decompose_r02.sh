mkdir -p gpurun_out/r02
for e in - norm qkv attn norm,qkv,attn; do
  if [ "$e" = "-" ]; then unset LP_DEBUG_EMPTY; else export LP_DEBUG_EMPTY=$e; fi
  timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 >> gpurun_out/r02/decompose32.txt 2>&1
done
unset LP_DEBUG_EMPTY
