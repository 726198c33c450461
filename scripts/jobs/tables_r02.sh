mkdir -p gpurun_out/r02
timeout 1500 python scripts/bucket_roofline.py qwen2.5-32b --long --long-h 0,1536,3584,6144 --depths 1,2,4,8,16 --out gpurun_out/r02/buckets_32b_final.json > gpurun_out/r02/buckets_32b_final.log 2>&1
timeout 1200 python scripts/bucket_roofline.py qwen2.5-7b --long --depths 1,2,4,8,16,32,64 --out gpurun_out/r02/buckets_7b_final.json > gpurun_out/r02/buckets_7b_final.log 2>&1
timeout 1500 python scripts/run_configs.py c2 c3 c4 > gpurun_out/r02/configs_final.log 2>&1
cp gpurun_out/configs.json gpurun_out/r02/configs_final.json 2>/dev/null
