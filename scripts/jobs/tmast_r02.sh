# TMA-store epilogue for fp32 partials: parity, timeline, whole-forward A/B vs the previous build.
mkdir -p gpurun_out/r02
o=gpurun_out/r02/tmast.txt
: > $o
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_forward_gpu.py -q -x 2>&1 | tail -2 >> $o
LP_PROF_ONLY=small python scripts/gemm_prof.py qwen2.5-7b 2>&1 | grep -E "qkv|  o |down" | sed -E 's/.*M=([0-9]+).*last acc -> epi done ([0-9.]+).*end med\/max ([0-9.\/]+) us/M=\1 epi \2 end \3/' >> $o
LP_PROF_ONLY=bucket python scripts/gemm_prof.py qwen2.5-32b 2>&1 | grep -E "qkv|  o |down" | sed -E 's/.*M=([0-9]+).*last acc -> epi done ([0-9.]+).*end med\/max ([0-9.\/]+) us/M=\1 epi \2 end \3/' >> $o
for M in qwen2.5-7b qwen2.5-32b; do
  for rep in 1 2; do
    LP_AB_MODEL=$M LP_LIB=build/ab/rn1.so timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
    LP_AB_MODEL=$M timeout 600 python scripts/ab_forward.py 15 >> $o 2>&1
  done
done
for rep in 1 2; do
  LP_LIB=build/ab/rn1.so timeout 600 python scripts/ab_bench.py c2 >> $o 2>&1
  timeout 600 python scripts/ab_bench.py c2 >> $o 2>&1
done
cat $o
