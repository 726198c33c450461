# Packed fp32x2 softmax (attn_tc.cu slice_exp_sum): kernel times per polynomial share.
mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/attn_pk*
for v in scalar_4_1 pk_8_3 pk_4_1 pk_8_2 pk_2_1 pk_8_1; do bash scripts/jobs/attn_r02.sh pk$v build/ab/sm_$v.so; done
python scripts/attn_table.py gpurun_out/r02/attn_pk*_qwen2.5-32b.csv gpurun_out/r02/attn_pk*_qwen2.5-7b.csv > gpurun_out/r02/softmax_pk.txt 2>&1
cat gpurun_out/r02/softmax_pk.txt
