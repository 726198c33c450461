mkdir -p gpurun_out/r02
export LP_PARITY_OUT=gpurun_out/r02/full_depth_parity3.jsonl
rm -f $LP_PARITY_OUT
timeout 1500 python -m pytest tests/test_full_depth_gpu.py -q > gpurun_out/r02/full_depth3.log 2>&1
echo "rc=$?" >> gpurun_out/r02/full_depth3.log
o=gpurun_out/r02/sanitizer2.txt
: > $o
for tool in memcheck synccheck racecheck; do
  echo "## $tool (scripts/sanitize_run2.py)" >> $o
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_run2.py >> $o 2>&1
  echo "rc=$?" >> $o
done
