"""Attention cost with long histories: 7B shape, 1 layer; a session is
prefilled to H tokens, then a chunk of C tokens runs at history H."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_11589_b200.instance import QWEN25_7B, Member, PrefillInstance, KIND_STANDARD
m = QWEN25_7B.with_layers(1)
inst = PrefillInstance(m, max_tokens=8192, max_members=64, kv_pages=4096, use_graphs=False)
rng = np.random.default_rng(0)
for H, C, nreq in ((4096, 512, 1), (8192, 512, 1), (2048, 128, 8), (0, 256, 16), (1024, 64, 32)):
    sids = list(range(1000 * H + C, 1000 * H + C + nreq))
    for s in sids:
        for p in range(0, H, 4096):
            n = min(4096, H - p)
            inst.forward(0, 0, 2, [Member(0, s, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))
    ts = []
    for it in range(5):
        ms = [Member(i, s, C, H) for i, s in enumerate(sids)]
        ts.append(inst.forward(0, 0, 2, ms, rng.integers(0, m.vocab, C * nreq).astype(np.int32)))
    fl = 4.0 * m.n_q_heads * m.head_dim * nreq * C * (H + (C + 1) / 2)
    t = float(np.median(ts[1:]))
    print(f"H={H:5d} C={C:4d} n={nreq:2d}: fwd {t:.3f} ms  attn flops {fl/1e9:.1f} GF", flush=True)
    for s in sids: inst.release(s)
