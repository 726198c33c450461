mkdir -p gpurun_out/r02
o=gpurun_out/r02/skprof.txt
: > $o
for v in 0 2; do
  echo "## LP_STREAMK=$v" >> $o
  LP_STREAMK=$v python scripts/gemm_prof.py qwen2.5-32b 2>&1 | sed -E 's/forward ([0-9.]+ ms).*pdl_wait returns ([0-9.]+).*first operands \+([0-9.]+).*MMA span ([0-9.]+) \(max ([0-9.]+)\).*last acc -> epi done ([0-9.]+).*end med\/max ([0-9.\/]+) us/fwd \1 | pdl \2 | first +\3 | mma \4 max \5 | epi \6 | end \7/' >> $o
done
cat $o
