mkdir -p gpurun_out/r02
o=gpurun_out/r02/ab_fuse.txt
: > $o
for rep in 1 2 3; do
  for f in none qkv resid 1; do
    if [ $f = none ]; then unset LP_FUSE_EPI; else export LP_FUSE_EPI=$f; fi
    echo -n "fuse=$f " >> $o
    timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  done
done
unset LP_FUSE_EPI
cat $o
