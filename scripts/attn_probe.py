"""Attention kernel probe for ncu: Qwen2.5-7B shape, 1 layer. A 512-token
long-prefill chunk (chunk graph, tcgen05 attention) at history H for each H
in argv, then a 16-token re-prefill at H=1024 (grid graph, warp-MMA kernel).
usage: attn_probe.py [H ...]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import (KIND_GRAPH, KIND_STANDARD, QWEN25_7B, Member,  # noqa: E402
                                            PrefillInstance)

m = QWEN25_7B.with_layers(1)
inst = PrefillInstance(m, max_tokens=4096, max_members=16, kv_pages=512)
inst.capture_graphs(lengths=(16,), depths=(1,))
rng = np.random.default_rng(0)
hs = [int(x) for x in sys.argv[1:]] or [0, 1536, 3584]


def fill(s, H):
    for p in range(0, H, 4096):
        n = min(4096, H - p)
        inst.forward(n, 1, KIND_STANDARD, [Member(0, s, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))


for i, H in enumerate(hs):
    s = 100 + i
    fill(s, H)
    for it in range(3):
        t = inst.forward(512, 1, KIND_STANDARD, [Member(1, s, 512, H)], rng.integers(0, m.vocab, 512).astype(np.int32))
    print(f"chunk 512 @ H={H}: {t:.3f} ms (1 layer)", flush=True)
fill(7, 1024)
for it in range(3):
    t = inst.forward(16, 1, KIND_GRAPH, [Member(2, 7, 16, 1024)], rng.integers(0, m.vocab, 16).astype(np.int32))
print(f"re-prefill 16 @ H=1024: {t:.3f} ms (1 layer)")
