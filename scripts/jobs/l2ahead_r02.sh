# L2 weight prefetch before the PDL wait: timeline + forward A/B.
mkdir -p gpurun_out/r02
o=gpurun_out/r02/l2ahead.txt
: > $o
for v in 0 1; do
  echo "## LP_L2_AHEAD=$v" >> $o
  LP_L2_AHEAD=$v python scripts/gemm_prof.py qwen2.5-32b 2>&1 | sed -E 's/forward ([0-9.]+ ms).*pdl_wait returns ([0-9.]+).*first operands \+([0-9.]+).*MMA span ([0-9.]+).*last acc -> epi done ([0-9.]+).*end med\/max ([0-9.\/]+) us/fwd \1 | pdl \2 | first +\3 | mma \4 | epi \5 | end \6/' >> $o
done
for rep in 1 2; do for v in 0 1; do
  echo "## chunk LP_L2_AHEAD=$v rep $rep" >> $o
  LP_L2_AHEAD=$v timeout 300 python scripts/decompose_chunk.py qwen2.5-32b 0 4096 2>&1 | grep chunk512 >> $o
done; done
cat $o
