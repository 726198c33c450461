mkdir -p gpurun_out/r02
tag=$1
ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 2 -c 1 -o gpurun_out/r02/attn_full_${tag} python scripts/attn_bench.py qwen2.5-32b 8192 > gpurun_out/r02/attn_full_${tag}.log 2>&1
ncu -i gpurun_out/r02/attn_full_${tag}.ncu-rep --page details --csv > gpurun_out/r02/attn_full_${tag}_details.csv 2>&1
ncu -i gpurun_out/r02/attn_full_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/r02/attn_full_${tag}_source.csv 2>&1
