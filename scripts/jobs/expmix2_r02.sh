mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/attn_x*
bash scripts/jobs/attn_r02.sh x_3_1
for v in 4_1 5_1 6_1 8_1 1_0 16_3; do bash scripts/jobs/attn_r02.sh x_$v build/ab/exp_$v.so; done
python scripts/attn_table.py gpurun_out/r02/attn_x_*_qwen2.5-32b.csv gpurun_out/r02/attn_x_*_qwen2.5-7b.csv > gpurun_out/r02/expmix2.txt 2>&1
cat gpurun_out/r02/expmix2.txt
