"""Sweep (token tiles, split-K) for one projection GEMM against the planner's
choice (LP_TIME_GEMM_PLAN override of Instance::time_gemm), CUDA events.
usage: tile_sweep.py MODEL WHICH T [T...]   (WHICH: 0 qkv, 1 o, 2 gate/up, 3 down)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import MODELS, PrefillInstance  # noqa: E402

model = MODELS[sys.argv[1]]
which = int(sys.argv[2])
ts = [int(x) for x in sys.argv[3:]]
inst = PrefillInstance(model.with_layers(1), max_tokens=max(max(ts), 512), max_members=64, kv_pages=64)
for t in ts:
    os.environ.pop("LP_TIME_GEMM_PLAN", None)
    base = inst.time_gemm(0, which, t, t, iters=50)
    res = []
    for nt in range(1, 9):
        for s in (1, 2, 3, 4, 5, 6, 8):
            os.environ["LP_TIME_GEMM_PLAN"] = f"{nt},{s}"
            res.append((inst.time_gemm(0, which, t, t, iters=50), nt, s))
    os.environ.pop("LP_TIME_GEMM_PLAN", None)
    res.sort()
    print(f"{sys.argv[1]} which={which} T={t}: planner {base * 1e3:.1f} us; best " +
          ", ".join(f"nt{nt}/s{s} {ms * 1e3:.1f}" for ms, nt, s in res[:8]), flush=True)
