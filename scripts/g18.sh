for f in 1 0; do echo "LP_FUSE_EPI=$f"; for s in "256 16" "256 64"; do LP_FUSE_EPI=$f timeout 300 python scripts/prof_forward.py $s; done; done
