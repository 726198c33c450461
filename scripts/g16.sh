K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 1160 -c 580 --csv --log-file gpurun_out/l32_512.csv python scripts/prof_forward.py 512 1 0 qwen2.5-32b > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 1040 -c 520 --csv --log-file gpurun_out/l7_512.csv python scripts/prof_forward.py 512 1 0 qwen2.5-7b > /dev/null 2>&1
