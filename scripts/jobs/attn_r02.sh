mkdir -p gpurun_out/r02
tag=${1:-cur}
[ -n "$2" ] && export LP_LIB=$2
for M in qwen2.5-32b qwen2.5-7b; do
  ncu --clock-control none -k regex:attn_tc --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02/attn_${tag}_${M}.csv python scripts/attn_bench.py $M > gpurun_out/r02/attn_${tag}_${M}.log 2>&1
done
