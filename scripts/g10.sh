make -s -C oracle synth
export LP_BENCH_QUICK=1
K='regex:gemm|attn|qkv|resid|embed|gather|argmax'
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py --steps 4 --warmup 3 > gpurun_out/ncu_bench_stdout.txt 2>&1
echo "launch list rc=$?"
ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/r01_gateup_full python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full_stdout.txt 2>&1
echo "full rc=$?"
tail -2 gpurun_out/ncu_bench_stdout.txt | cut -c1-400
