mkdir -p gpurun_out/r02
o=gpurun_out/r02/sk_ab2.txt
: > $o
for rep in 1 2 3; do for v in 0 1 2; do
  echo "## LP_STREAMK=$v rep $rep" >> $o
  LP_STREAMK=$v timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 2048 4096 2>&1 | grep chunk512 >> $o
done; done
for v in 0 1 2; do
  echo "## 7B LP_STREAMK=$v" >> $o
  LP_STREAMK=$v timeout 300 python scripts/decompose_chunk.py qwen2.5-7b 0 4096 2>&1 | grep chunk512 >> $o
done
cat $o
