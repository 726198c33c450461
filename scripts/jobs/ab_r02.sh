# A/B the previous build (build/ab/liblaps_old.so) against the current one on c2 and c4.
mkdir -p gpurun_out/r02
o=gpurun_out/r02/ab_bench.txt
: > $o
for rep in 1 2; do
  LP_LIB=build/ab/liblaps_old.so timeout 600 python scripts/ab_bench.py c2 >> $o 2>&1
  timeout 600 python scripts/ab_bench.py c2 >> $o 2>&1
done
for rep in 1 2; do
  LP_LIB=build/ab/liblaps_old.so timeout 600 python scripts/ab_bench.py c4 40 >> $o 2>&1
  timeout 600 python scripts/ab_bench.py c4 40 >> $o 2>&1
done
cat $o
