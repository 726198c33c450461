mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_forward_gpu.py -x -q > gpurun_out/r02/qpref_test.log 2>&1; echo "rc=$?" >> gpurun_out/r02/qpref_test.log
bash scripts/jobs/attn_r02.sh qpref
bash scripts/jobs/attn_r02.sh persist1b build/ab/persist1.so
