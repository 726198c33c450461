for N in 190 300 700 1500; do
  for bn in 128 256; do
    python scripts/gemm_one.py 37888 $N 3584 2 $bn 2 1 10
    for s in 1 2 3; do python scripts/gemm_one.py 3584 $N 18944 1 $bn 2 $s 10; done
  done
done 2>&1 | grep -v "^ \|Exception\|Traceback\|ModuleNotFound"
