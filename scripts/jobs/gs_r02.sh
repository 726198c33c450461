mkdir -p gpurun_out/r02
o=gpurun_out/r02/gs.txt
: > $o
timeout 900 python -m pytest tests/test_forward_gpu.py -q -x 2>&1 | tail -1 >> $o
python scripts/kernel_timeline.py qwen2.5-32b chunk 0 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-32b bucket 256 1 >> $o 2>&1
for M in qwen2.5-32b qwen2.5-7b; do
  for rep in 1 2; do
    LP_AB_MODEL=$M LP_LIB=build/ab/rn1.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
    LP_AB_MODEL=$M timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  done
done
cat $o
