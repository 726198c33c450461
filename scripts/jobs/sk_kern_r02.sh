# Per-kernel durations of a full-depth 32B 512-token chunk (H=2048) with split-K vs forced stream-K plans.
mkdir -p gpurun_out/r02
for v in 1 2 0; do
  LP_STREAMK=$v ncu --nvtx --nvtx-include target/ --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02/skk_$v.csv python scripts/ncu_forward.py qwen2.5-32b standard 512 1 2048 > gpurun_out/r02/skk_$v.log 2>&1
  echo "== LP_STREAMK=$v"; python scripts/summarize_ncu.py gpurun_out/r02/skk_$v.csv | head -12
done
