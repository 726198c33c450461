mkdir -p gpurun_out/r02
o=gpurun_out/r02/kernel_timeline.txt
: > $o
python scripts/kernel_timeline.py qwen2.5-7b bucket 16 1 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-7b bucket 256 1 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-32b bucket 16 1 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-32b bucket 256 1 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-32b chunk 0 >> $o 2>&1
python scripts/kernel_timeline.py qwen2.5-32b chunk 4096 >> $o 2>&1
cat $o
