# Fraction of softmax exponentials on the FMA pipe (attn_tc.cu kExpFmaMod / kExpFmaCnt): kernel times.
mkdir -p gpurun_out/r02
bash scripts/jobs/attn_r02.sh exp_3_1
for v in 2_1 5_2 8_3 16_7 4_1; do bash scripts/jobs/attn_r02.sh exp_$v build/ab/exp_$v.so; done
bash scripts/jobs/attn_r02.sh exp_3_1b
python scripts/attn_table.py gpurun_out/r02/attn_exp_*_qwen2.5-32b.csv gpurun_out/r02/attn_exp_*_qwen2.5-7b.csv > gpurun_out/r02/expmix.txt 2>&1
cat gpurun_out/r02/expmix.txt
