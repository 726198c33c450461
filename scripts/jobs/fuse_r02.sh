mkdir -p gpurun_out/r02
out=gpurun_out/r02/fuse.txt
for M in qwen2.5-32b qwen2.5-7b; do
for f in 0 qkv resid 1 0; do
  LP_FUSE_EPI=$f timeout 300 python scripts/decompose_chunk.py $M 0 4096 2>&1 | grep chunk512 | sed "s/^/fuse=$f /" >> $out
done
done
