"""A/B timing of a 7B 512-token long-prefill chunk at history H with a given
build of the native library (experiments: compare two kernel variants on the
same box back to back). usage: ab_chunk.py LIB_PATH [H] [ITERS]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402

N.LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2601_11589_b200.instance import KIND_STANDARD, QWEN25_7B, Member, PrefillInstance  # noqa: E402

H = int(sys.argv[2]) if len(sys.argv) > 2 else 3584
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 7
m = QWEN25_7B
inst = PrefillInstance(m, max_tokens=4096, max_members=8, kv_pages=256)
inst.capture_graphs(lengths=(16,), depths=(1,))
rng = np.random.default_rng(0)
ts = []
for it in range(iters + 2):
    s = 10 + it
    if H:
        inst.forward(H, 1, KIND_STANDARD, [Member(0, s, H, 0)], rng.integers(0, m.vocab, H).astype(np.int32))
    t = inst.forward(512, 1, KIND_STANDARD, [Member(0, s, 512, H)], rng.integers(0, m.vocab, 512).astype(np.int32))
    if it >= 2:
        ts.append(t)
    inst.release(s)
print(f"{N.LIB_PATH.parent.name}: chunk 512 at H={H}: median {np.median(ts):.3f} ms  min {min(ts):.3f}")
