# Packed softmax in the product build: GPU suite (incl. full depth), attention table, c4 A/B vs the previous build.
mkdir -p gpurun_out/r02
export LP_PARITY_OUT=gpurun_out/r02/full_depth_parity_pk.jsonl
rm -f $LP_PARITY_OUT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02/gputest_pk.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gputest_pk.log
tail -2 gpurun_out/r02/gputest_pk.log
rm -f gpurun_out/r02/attn_final*
bash scripts/jobs/attn_r02.sh final
python scripts/attn_table.py gpurun_out/r02/attn_final_qwen2.5-32b.csv gpurun_out/r02/attn_final_qwen2.5-7b.csv > gpurun_out/r02/attn_final.txt 2>&1
cat gpurun_out/r02/attn_final.txt
o=gpurun_out/r02/ab_pk.txt
: > $o
for rep in 1 2; do
  LP_LIB=build/ab/liblaps_old.so timeout 600 python scripts/ab_bench.py c4 40 >> $o 2>&1
  timeout 600 python scripts/ab_bench.py c4 40 >> $o 2>&1
done
cat $o
