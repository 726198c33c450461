K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 600 -c 300 --csv --log-file gpurun_out/l7_256x16_b.csv python scripts/prof_forward.py 256 16 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 600 -c 300 --csv --log-file gpurun_out/l7_16x1_b.csv python scripts/prof_forward.py 16 1 > /dev/null 2>&1
