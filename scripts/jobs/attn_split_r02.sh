mkdir -p gpurun_out/r02
for f in 1 2 3 4; do
  export LP_ATTN_TC_SPLIT=$f
  for M in qwen2.5-32b qwen2.5-7b; do
    ncu --clock-control none -k regex:attn_tc --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02/attn_split${f}_${M}.csv python scripts/attn_bench.py $M 0 2048 3584 8192 > gpurun_out/r02/attn_split${f}_${M}.log 2>&1
  done
  timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 2>&1 | grep chunk512 | sed "s/^/split=$f /" >> gpurun_out/r02/attn_split_fwd.txt
done
