"""Where a long-prompt chunk forward's time goes (event-timed, not under a
profiler): median ms of a C_l = 512-token chunk (chunk graph) over histories
H, plus each projection GEMM alone (time_gemm, same launch plan). Run it with
LP_DEBUG_EMPTY=norm / qkv / attn / norm,qkv,attn to replace those kernels by
empty PDL launches (timing decomposition only; the results are wrong).
usage: decompose_chunk.py MODEL [H ...]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

name = sys.argv[1]
Hs = [int(x) for x in sys.argv[2:]] or [0, 4096]
m = MODELS[name]
inst = PrefillInstance(m, max_tokens=4096, max_members=8, kv_pages=512)
inst.capture_graphs(lengths=(64,), depths=(1,))
rng = np.random.default_rng(0)
tag = os.environ.get("LP_DEBUG_EMPTY", "-")
sid = 1
for H in Hs:
    ts = []
    for it in range(5):
        done = 0
        while done < H:
            c = min(4096, H - done)
            inst.forward(c, 1, KIND_STANDARD, [Member(0, sid, c, done)], rng.integers(0, m.vocab, c).astype(np.int32))
            done += c
        ts.append(inst.forward(512, 1, KIND_STANDARD, [Member(1, sid, 512, H)],
                               rng.integers(0, m.vocab, 512).astype(np.int32)))
        inst.release(sid)
        sid += 1
    print(f"{name} empty={tag} chunk512 H={H}: {np.median(ts[1:]):.3f} ms", flush=True)
if tag == "-":
    for which, nm in enumerate(["qkv", "o", "gate_up", "down"]):
        us = inst.time_gemm(0, which, 512, 512, iters=20) * 1e3
        print(f"{name} gemm {nm} t=512: {us:.1f} us x {m.layers} layers = {us * m.layers / 1e3:.2f} ms", flush=True)
