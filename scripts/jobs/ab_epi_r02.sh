mkdir -p gpurun_out/r02
o=gpurun_out/r02/ab_epi2.txt
: > $o
for rep in 1 2 3; do
  LP_LIB=build/ab/liblaps_old.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  LP_LIB=build/ab/epi1.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  LP_LIB=build/ab/epi2.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
done
cat $o
