"""Sweep (token tiles, split-K) for one projection GEMM against the planner's
choice (LP_TIME_GEMM_PLAN override of Instance::time_gemm), CUDA events.
usage: tile_sweep.py WHICH T [T...]   (WHICH: 0 qkv, 1 o, 2 gate/up, 3 down)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import QWEN25_7B, PrefillInstance  # noqa: E402

which = int(sys.argv[1])
ts = [int(x) for x in sys.argv[2:]]
inst = PrefillInstance(QWEN25_7B.with_layers(1), max_tokens=max(ts), max_members=64, kv_pages=64)
for t in ts:
    os.environ.pop("LP_TIME_GEMM_PLAN", None)
    base = inst.time_gemm(0, which, t, t, iters=50)
    res = []
    for nt in (1, 2, 3, 4):
        for s in (1, 2, 3, 4, 6, 8):
            os.environ["LP_TIME_GEMM_PLAN"] = f"{nt},{s}"
            res.append((inst.time_gemm(0, which, t, t, iters=50), nt, s))
    res.sort()
    print(f"which={which} T={t}: planner {base * 1e3:.1f} us; best " +
          ", ".join(f"nt{nt}/s{s} {ms * 1e3:.1f}" for ms, nt, s in res[:6]), flush=True)
