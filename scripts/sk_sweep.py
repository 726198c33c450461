"""Stream-K vs the best split-K plan per projection (LP_TIME_GEMM_PLAN
overrides of Instance::time_gemm, CUDA events, 50 iterations each).
usage: sk_sweep.py MODEL"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import MODELS, PrefillInstance  # noqa: E402

model = MODELS[sys.argv[1]]
inst = PrefillInstance(model.with_layers(1), max_tokens=4096, max_members=64, kv_pages=64)
names = {0: "qkv", 1: "o", 3: "down"}


def timed(which, t, plan=None):
    if plan is None:
        os.environ.pop("LP_TIME_GEMM_PLAN", None)
    else:
        os.environ["LP_TIME_GEMM_PLAN"] = plan
    inst.time_gemm(0, which, t, t, iters=5)
    return inst.time_gemm(0, which, t, t, iters=50) * 1e3


for which in (0, 1, 3):
    for t in (256, 384, 512, 1024, 2048):
        planner = timed(which, t)
        best_split = min((timed(which, t, f"{nt},{s}"), nt, s) for nt in range(1, 9) for s in (1, 2, 3, 4, 5, 6, 8))
        sk = sorted((timed(which, t, f"{nt},-1"), nt) for nt in range(1, 9))
        print(f"{sys.argv[1]} {names[which]} T={t}: planner {planner:.1f} us; best split nt{best_split[1]}/s{best_split[2]} "
              f"{best_split[0]:.1f}; stream-K " + ", ".join(f"nt{nt} {us:.1f}" for us, nt in sk[:4]), flush=True)
os.environ.pop("LP_TIME_GEMM_PLAN", None)
