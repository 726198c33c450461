mkdir -p gpurun_out/r02
o=gpurun_out/r02/ab_fwd.txt
: > $o
for rep in 1 2 3; do
  LP_LIB=build/ab/liblaps_old.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
done
cat $o
