for n in 1024 2048 4096; do python scripts/gemm_one.py 37888 $n 3584 2 256 2 1 10; done
python scripts/gemm_one.py 37888 256 3584 2 256 2 1 10
ncu --set full --clock-control none -k regex:gemm -s 2 -c 1 -o gpurun_out/gu1024 python scripts/gemm_one.py 37888 1024 3584 2 256 2 1 3 > /dev/null 2>&1
ncu -i gpurun_out/gu1024.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for i,n in enumerate(h):
    if n in ('gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'): print(n, v[i], r[1][i])
"
