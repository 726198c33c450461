# Refresh the dominant-kernel ncu capture on the final code (gate/up + SiLU, 32B, 512-token chunk).
mkdir -p gpurun_out/r02
ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/r02/gu32_512_final python scripts/prof_dominant.py 512 512 3 2 qwen2.5-32b > gpurun_out/r02/gu32_final.log 2>&1
ncu -i gpurun_out/r02/gu32_512_final.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__cycles_active.avg,sm__cycles_elapsed.avg > gpurun_out/r02/gu32_final_raw.csv 2>&1
cat gpurun_out/r02/gu32_final_raw.csv | tail -3
