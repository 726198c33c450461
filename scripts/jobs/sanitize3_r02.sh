# Sanitizer pass for this session's kernels + the TMEM pair-alloc racecheck repro.
mkdir -p gpurun_out/r02
o=gpurun_out/r02/sanitizer3.txt
: > $o
for v in 0 1; do
  echo "## racecheck build/repro_tmem $v (scripts/repro/racecheck_tmem_alloc_pair.cu)" >> $o
  timeout 300 compute-sanitizer --tool racecheck build/repro_tmem $v >> $o 2>&1
  echo "rc=$?" >> $o
done
for tool in memcheck synccheck; do
  echo "## $tool: stream-K / split-K GEMMs (tests/test_gemm_gpu.py -k 'stream_k or splitk or pair')" >> $o
  timeout 1200 compute-sanitizer --tool $tool python -m pytest tests/test_gemm_gpu.py -q -k "stream_k or splitk or pair" >> $o 2>&1
  echo "rc=$?" >> $o
done
for tool in memcheck synccheck racecheck; do
  echo "## $tool: packed-softmax tcgen05 attention (tests/test_forward_gpu.py -k 'persistent or tc')" >> $o
  timeout 1500 compute-sanitizer --tool $tool python -m pytest tests/test_forward_gpu.py -q -k "persistent" >> $o 2>&1
  echo "rc=$?" >> $o
done
grep -E "^##|ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=|variant" $o
