# Persistent attention with 4 softmax groups (576 threads) vs 2: parity + kernel times.
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_forward_gpu.py -q -x > gpurun_out/r02/sg_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02/sg_test.log
tail -2 gpurun_out/r02/sg_test.log
rm -f gpurun_out/r02/attn_sg*
bash scripts/jobs/attn_r02.sh sg2 build/ab/sg2.so
bash scripts/jobs/attn_r02.sh sg4 build/ab/sg4.so
bash scripts/jobs/attn_r02.sh sg2b build/ab/sg2.so
python scripts/attn_table.py gpurun_out/r02/attn_sg*_qwen2.5-32b.csv gpurun_out/r02/attn_sg*_qwen2.5-7b.csv > gpurun_out/r02/sg.txt 2>&1
cat gpurun_out/r02/sg.txt
