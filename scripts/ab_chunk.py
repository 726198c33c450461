"""A/B timing of one forward shape with a given build of the native library
(experiments: compare two kernel variants on the same box back to back).
usage: ab_chunk.py LIB_PATH chunk H [ITERS]
       ab_chunk.py LIB_PATH graph L_PAD DEPTH H [ITERS]   (AB_MODEL, default qwen2.5-7b; members L ~ U(l_pad/2+1, l_pad))"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402

N.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

mode = sys.argv[2]
import os
m = MODELS[os.environ.get("AB_MODEL", "qwen2.5-7b")]
rng = np.random.default_rng(0)
if mode == "chunk":
    lp, dp, H = 512, 1, int(sys.argv[3])
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 7
else:
    lp, dp, H = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 7
inst = PrefillInstance(m, max_tokens=max(4096, lp * dp), max_members=max(8, dp), kv_pages=max(256, dp * (H + lp) // 64 + 64))
inst.capture_graphs(lengths=(lp if mode == "graph" else 16,), depths=(dp if mode == "graph" else 1,))
ts, sid = [], 10
for it in range(iters + 2):
    ms = []
    for i in range(dp):
        sid += 1
        for p in range(0, H, 4096):
            n = min(4096, H - p)
            inst.forward(n, 1, KIND_STANDARD, [Member(0, sid, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))
        L = lp if mode == "chunk" else int(rng.integers(lp // 2 + 1, lp + 1))
        ms.append(Member(i, sid, L, H))
    toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in ms)).astype(np.int32)
    t = inst.forward(lp, dp, KIND_STANDARD if mode == "chunk" else KIND_GRAPH, ms, toks)
    if it >= 2:
        ts.append(t)
    for x in ms:
        inst.release(x.session_id)
print(f"{N.LIB_PATH.parent.name}: {mode} {lp}x{dp} H={H}: median {np.median(ts):.3f} ms  min {min(ts):.3f}")
