for s in "256 1" "16 1" "128 8"; do python scripts/prof_forward.py $s; done
K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
# skip the eager warm-up forward + 2 replays (256 launches each for 28 layers), profile one replay
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 768 -c 256 --csv --log-file gpurun_out/l_256x1.csv python scripts/prof_forward.py 256 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 768 -c 256 --csv --log-file gpurun_out/l_16x1.csv python scripts/prof_forward.py 16 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 768 -c 256 --csv --log-file gpurun_out/l_128x8.csv python scripts/prof_forward.py 128 8 > /dev/null 2>&1
echo done
