set -x
mkdir -p gpurun_out/r02
ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/r02/gu32_512 python scripts/prof_dominant.py 512 512 3 2 qwen2.5-32b > gpurun_out/r02/gu32.log 2>&1
ncu -i gpurun_out/r02/gu32_512.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second > gpurun_out/r02/gu32_raw.csv 2>&1
ncu --nvtx --nvtx-include target/ --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/r02/chunk32_h8192.csv python scripts/ncu_forward.py qwen2.5-32b standard 512 1 8192 > gpurun_out/r02/chunk32.log 2>&1
python scripts/summarize_ncu.py gpurun_out/r02/chunk32_h8192.csv > gpurun_out/r02/chunk32_summary.txt 2>&1
LP_BENCH_OUT=gpurun_out/r02/bench_run python bench.py --steps 40 --warmup 5 > gpurun_out/r02/bench40.json 2>gpurun_out/r02/bench40.err
