mkdir -p gpurun_out/r02
o=gpurun_out/r02/ab_st.txt
: > $o
for M in qwen2.5-7b qwen2.5-32b; do
  for rep in 1 2; do
    for v in st8 st10 st6; do
      LP_AB_MODEL=$M LP_LIB=build/ab/$v.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
    done
  done
done
cat $o
