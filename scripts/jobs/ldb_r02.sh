mkdir -p gpurun_out/r02
rm -f gpurun_out/r02/attn_ldb* gpurun_out/r02/attn_cur*
bash scripts/jobs/attn_r02.sh cur build/ab/cur.so
bash scripts/jobs/attn_r02.sh ldb build/ab/ldb.so
bash scripts/jobs/attn_r02.sh cur2 build/ab/cur.so
python scripts/attn_table.py gpurun_out/r02/attn_cur_*.csv gpurun_out/r02/attn_ldb_*.csv gpurun_out/r02/attn_cur2_*.csv
