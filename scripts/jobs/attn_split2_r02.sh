mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests/test_forward_gpu.py -x -q > gpurun_out/r02/split2_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02/split2_test.log
for f in 1 2 3 4; do
  export LP_ATTN_TC_SPLIT=$f
  for M in qwen2.5-32b qwen2.5-7b; do
    ncu --clock-control none -k regex:attn_tc --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02/attn_s2split${f}_${M}.csv python scripts/attn_bench.py $M 0 2048 3584 8192 > gpurun_out/r02/attn_s2split${f}_${M}.log 2>&1
  done
done
