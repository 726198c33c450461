"""Long-prompt attention micro-benchmark: one decoder layer of MODEL; a
session is prefilled to H tokens, then a C-token chunk runs at history H
(eager standard launch -> the tcgen05 attention kernel). Run under
  ncu -k regex:attn_tc --metrics gpu__time_duration.sum --csv --log-file X python scripts/attn_bench.py MODEL
and read the attn_tc_kernel launches (3 per config, the last two warm);
prints the causal attention flops per config: 4 nq d C (H + (C+1)/2).
usage: attn_bench.py MODEL [H ...]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402

from paper_2601_11589_b200 import _native as N  # noqa: E402

if os.environ.get("LP_LIB"):  # A/B: another build of the native library
    N.LIB_PATH = Path(os.environ["LP_LIB"]).resolve()
from paper_2601_11589_b200.instance import KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

m = MODELS[sys.argv[1]].with_layers(1)
Hs = [int(x) for x in sys.argv[2:]] or [0, 2048, 3584, 8192, 16384]
C = 512
inst = PrefillInstance(m, max_tokens=8192, max_members=8, kv_pages=1024, use_graphs=False)
rng = np.random.default_rng(0)
for H in Hs:
    sid = 100 + H
    for p in range(0, H, 8192):
        n = min(8192, H - p)
        inst.forward(n, 1, KIND_STANDARD, [Member(0, sid, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))
    for it in range(3):
        inst.forward(C, 1, KIND_STANDARD, [Member(1, sid, C, H)], rng.integers(0, m.vocab, C).astype(np.int32))
    fl = 4.0 * m.n_q_heads * m.head_dim * C * (H + (C + 1) / 2)
    print(f"{sys.argv[1]} H={H} C={C}: attention {fl / 1e9:.2f} GFLOP per layer", flush=True)
    inst.release(sid)
