"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): graph
replays, an eager long chunk (tcgen05 attention with in-kernel merge), a
re-prefill over resident history (split-KV + merge grid) and a session
migration, on the tiny model and a 2-layer Qwen2.5-7B-shaped model.
usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import (KIND_GRAPH, KIND_STANDARD, QWEN25_7B, TINY, Member,  # noqa: E402
                                            PrefillInstance)

rng = np.random.default_rng(0)
for m in (TINY, QWEN25_7B.with_layers(2)):
    a = PrefillInstance(m, max_tokens=1024, max_members=8, kv_pages=64)
    b = PrefillInstance(m, max_tokens=1024, max_members=8, kv_pages=64)
    a.capture_graphs(lengths=(16, 64), depths=(1, 4))
    tok = lambda n: rng.integers(0, m.vocab, n).astype(np.int32)  # noqa: E731
    a.forward(64, 4, KIND_GRAPH, [Member(0, 1, 50, 0), Member(1, 2, 33, 0), Member(2, 3, 64, 0)], tok(147))
    a.forward(512, 1, KIND_STANDARD, [Member(0, 4, 512, 0)], tok(512))          # long chunk, H = 0
    a.forward(300, 1, KIND_STANDARD, [Member(0, 4, 300, 512)], tok(300))        # next chunk over history
    a.forward(16, 4, KIND_GRAPH, [Member(0, 4, 9, 812), Member(1, 1, 16, 50)], tok(25))  # re-prefill
    PrefillInstance.migrate(a, b, 4)
    b.forward(16, 1, KIND_GRAPH, [Member(0, 4, 12, 821)], tok(12))
    print(m.name if hasattr(m, "name") else "model", "ok", a.next_tokens()[:2], b.next_tokens()[:1], flush=True)
    a.close()
    b.close()
