mkdir -p gpurun_out/r02
tag=$1
timeout 600 python -m pytest tests/test_forward_gpu.py -x -q -k "tcgen05 or long_history or deep_reprefill or 7b_shaped or 32b_shaped" > gpurun_out/r02/attn_test_${tag}.log 2>&1
echo "rc=$?" >> gpurun_out/r02/attn_test_${tag}.log
bash scripts/jobs/attn_r02.sh $tag
