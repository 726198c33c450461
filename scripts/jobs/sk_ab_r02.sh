# A/B: 32B / 7B chunk forwards with and without stream-K plans.
mkdir -p gpurun_out/r02
o=gpurun_out/r02/sk_ab.txt
: > $o
for rep in 1 2; do
  for sk in 0 1; do
    echo "## LP_STREAMK=$sk rep $rep" >> $o
    LP_STREAMK=$sk timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 >> $o 2>&1
  done
done
for sk in 0 1; do
  echo "## 7B LP_STREAMK=$sk" >> $o
  LP_STREAMK=$sk timeout 300 python scripts/decompose_chunk.py qwen2.5-7b 0 4096 >> $o 2>&1
done
cat $o
