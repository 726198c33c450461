mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/attn_deg*
for v in deg5 deg4 deg3 deg4_83b deg3_2; do bash scripts/jobs/attn_r02.sh $v build/ab/$v.so; done
python scripts/attn_table.py gpurun_out/r02/attn_deg*_qwen2.5-32b.csv gpurun_out/r02/attn_deg*_qwen2.5-7b.csv > gpurun_out/r02/deg.txt
cat gpurun_out/r02/deg.txt
