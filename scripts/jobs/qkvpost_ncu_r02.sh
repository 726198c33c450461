mkdir -p gpurun_out/r02
ncu --set full --import-source on --clock-control none -k regex:qkv_post -s 70 -c 1 -o gpurun_out/r02/qkvpost_full python scripts/ncu_forward.py qwen2.5-32b standard 512 1 0 > gpurun_out/r02/qkvpost_full.log 2>&1
ncu -i gpurun_out/r02/qkvpost_full.ncu-rep --page details --csv > gpurun_out/r02/qkvpost_details.csv 2>&1
ncu -i gpurun_out/r02/qkvpost_full.ncu-rep --page source --csv > gpurun_out/r02/qkvpost_source.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:resid_rmsnorm -s 140 -c 1 -o gpurun_out/r02/norm_full python scripts/ncu_forward.py qwen2.5-32b standard 512 1 0 > gpurun_out/r02/norm_full.log 2>&1
ncu -i gpurun_out/r02/norm_full.ncu-rep --page details --csv > gpurun_out/r02/norm_details.csv 2>&1
