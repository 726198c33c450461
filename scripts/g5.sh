make -s -C oracle synth
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_forward_gpu.py -x -q 2>&1 | tail -5
for s in "256 1" "16 1" "128 8" "256 64"; do python scripts/prof_forward.py $s; done
LP_PDL=0 python scripts/prof_forward.py 16 1
K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 768 -c 256 --csv --log-file gpurun_out/l2_16x1.csv python scripts/prof_forward.py 16 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 768 -c 256 --csv --log-file gpurun_out/l2_256x1.csv python scripts/prof_forward.py 256 1 > /dev/null 2>&1
