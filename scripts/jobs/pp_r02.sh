# FA4-style ping-pong persistent attention (LP_ATTN_PINGPONG=1): parity + kernel times vs the shipped kernel.
mkdir -p gpurun_out/r02
LP_ATTN_PINGPONG=1 timeout 900 python -m pytest tests/test_forward_gpu.py -q -x > gpurun_out/r02/pp_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pp_test.log
tail -15 gpurun_out/r02/pp_test.log
rm -f gpurun_out/r02/attn_pp* gpurun_out/r02/attn_base4*
bash scripts/jobs/attn_r02.sh base4
LP_ATTN_PINGPONG=1 bash scripts/jobs/attn_r02.sh pp
python scripts/attn_table.py gpurun_out/r02/attn_base4_*.csv gpurun_out/r02/attn_pp_*.csv
