K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 480 -c 240 --csv --log-file gpurun_out/l7_256x16.csv python scripts/prof_forward.py 256 16 > /dev/null 2>&1
