for mode in 0 1 2 3; do python scripts/gemm_one.py 37888 2048 3584 $mode 256 2 1 10; done
python scripts/gemm_one.py 37888 2048 3584 2 256 1 1 10
python scripts/gemm_one.py 37888 2048 3584 2 128 2 1 10
python scripts/gemm_one.py 37888 2048 18944 2 256 2 1 5
python scripts/gemm_one.py 37888 2048 18944 0 256 2 1 5
ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/prof_silu python scripts/gemm_one.py 37888 2048 3584 2 256 2 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/prof_bf16 python scripts/gemm_one.py 37888 2048 3584 0 256 2 1 3 > /dev/null 2>&1
ls -la gpurun_out/
