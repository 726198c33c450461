make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for f in 1 0; do echo "LP_FUSE_EPI=$f"; for s in "256 16" "512 1" "256 64"; do LP_FUSE_EPI=$f timeout 300 python scripts/prof_forward.py $s; done; done
python scripts/gemm_plans.py qwen2.5-7b 16,256,512,2048
