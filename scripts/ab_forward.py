"""Per-forward A/B of two native-library builds (LP_LIB) on the 32B shape:
512-token chunks at several histories and a few graph buckets, median of N
event-timed forwards each (lp_submit/lp_wait), after warm-up.
usage: LP_LIB=... ab_forward.py [ITERS]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402

if os.environ.get("LP_LIB"):
    N.LIB_PATH = Path(os.environ["LP_LIB"]).resolve()
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 15
m = MODELS[os.environ.get("LP_AB_MODEL", "qwen2.5-32b")]
inst = PrefillInstance(m, max_tokens=8192, max_members=64, kv_pages=2048)
inst.capture_graphs()
rng = np.random.default_rng(0)
lib = Path(os.environ.get("LP_LIB", "product")).name
out = []


def timed(label, l_pad, kind, members, prep=None):
    toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in members)).astype(np.int32)
    ts = []
    for it in range(iters + 3):
        if prep:
            prep()
        ts.append(inst.forward(l_pad, len(members), kind, members, toks))
        for x in members:
            if x.history == 0:
                inst.release(x.session_id)
    out.append((label, float(np.median(ts[3:]))))


for H in (0, 2048, 4096):
    sid = 10 + H
    if H:
        inst.forward(H, 1, KIND_STANDARD, [Member(0, sid, H, 0)], rng.integers(0, m.vocab, H).astype(np.int32))
    timed(f"chunk512 H={H}", 512, KIND_STANDARD, [Member(1, sid if H else 9, 512, H)])
    inst.release(sid)
for l_pad, depth in ((16, 1), (128, 1), (256, 1), (64, 4), (32, 16)):
    mem = [Member(i, 1000 + i, int(rng.integers(l_pad // 2 + 1, l_pad + 1)), 0) for i in range(depth)]
    timed(f"graph {l_pad}x{depth}", l_pad, KIND_GRAPH, mem)
inst.close()
print(lib + " | " + " | ".join(f"{k} {v:.3f}" for k, v in out), flush=True)
