mkdir -p gpurun_out/r02
for w in 0 1 3; do
  timeout 300 python scripts/tile_sweep.py qwen2.5-32b $w 512 384 256 128 >> gpurun_out/r02/tiles32.txt 2>&1
  timeout 300 python scripts/tile_sweep.py qwen2.5-7b $w 512 384 256 >> gpurun_out/r02/tiles7.txt 2>&1
done
