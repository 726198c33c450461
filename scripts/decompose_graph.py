"""Where a graph-bucket forward's time goes (event-timed): median ms of an
(l_pad x depth) graph replay with members of L ~ U(l_pad/2, l_pad] at history H,
plus each projection GEMM alone at that live token count (time_gemm). Run with
LP_DEBUG_EMPTY=norm / qkv / attn to replace those kernels by empty PDL
launches (timing decomposition only; results wrong).
usage: decompose_graph.py MODEL L_PAD DEPTH [H]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

name, lp, dp = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
H = int(sys.argv[4]) if len(sys.argv) > 4 else 0
m = MODELS[name]
inst = PrefillInstance(m, max_tokens=max(4096, lp * dp), max_members=max(dp, 8), kv_pages=max(512, dp * (H + lp) // 64 + 64))
inst.capture_graphs(lengths=(lp,), depths=(dp,))
rng = np.random.default_rng(1)
tag = os.environ.get("LP_DEBUG_EMPTY", "-")
sid = 1
ts, T = [], 0
for it in range(7):
    ms = []
    for i in range(dp):
        done = 0
        while done < H:
            c = min(4096, H - done)
            inst.forward(c, 1, KIND_STANDARD, [Member(0, sid, c, done)], rng.integers(0, m.vocab, c).astype(np.int32))
            done += c
        ms.append(Member(i, sid, int(rng.integers(lp // 2 + 1, lp + 1)) if lp > 8 else lp, H))
        sid += 1
    T = sum(x.new_tokens for x in ms)
    ts.append(inst.forward(lp, dp, KIND_GRAPH, ms, rng.integers(0, m.vocab, T).astype(np.int32)))
    for x in ms:
        inst.release(x.session_id)
print(f"{name} empty={tag} graph {lp}x{dp} H={H} (T~{T}): {np.median(ts[2:]):.3f} ms", flush=True)
if tag == "-":
    for which, nm in enumerate(["qkv", "o", "gate_up", "down"]):
        us = inst.time_gemm(0, which, lp * dp, T, iters=20) * 1e3
        print(f"{name} gemm {nm} t_cap={lp * dp} n={T}: {us:.1f} us x {m.layers} = {us * m.layers / 1e3:.2f} ms", flush=True)
