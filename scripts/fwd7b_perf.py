"""Full-depth Qwen2.5-7B forward timing per graph shape (CUDA events via lp_wait)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2601_11589_b200.instance import QWEN25_7B, Member, PrefillInstance, KIND_GRAPH, KIND_STANDARD
cfg = QWEN25_7B
t0 = time.time()
inst = PrefillInstance(cfg, max_tokens=16384, max_members=64, kv_pages=4096)
print("create", time.time() - t0, flush=True)
shapes = [(256, 1), (128, 1), (64, 1), (16, 1), (256, 2), (128, 8), (256, 8), (256, 32), (256, 64)]
t0 = time.time()
inst.capture_graphs(lengths=sorted({s[0] for s in shapes}), depths=sorted({s[1] for s in shapes}))
print("capture", time.time() - t0, flush=True)
rng = np.random.default_rng(0)
sid = 0
W = 6.526e9 * 2 + 2 * 152064 * 3584
for (lp, dp) in shapes + [(512, 1)]:
    ts = []
    for it in range(6):
        ms = []
        for i in range(dp):
            L = int(rng.integers(max(1, lp // 2 + 1), lp + 1)) if lp > 8 else lp
            ms.append(Member(sid, sid, L, 0)); sid += 1
        toks = rng.integers(0, cfg.vocab, sum(m.new_tokens for m in ms)).astype(np.int32)
        kind = KIND_STANDARD if lp == 512 else KIND_GRAPH
        ts.append(inst.forward(lp, dp, kind, ms, toks))
        for m in ms: inst.release(m.session_id)
    t = float(np.median(ts[2:]))
    T = sum(m.new_tokens for m in ms)
    fl = 2 * 6.526e9 * T
    print(f"shape {lp:3d}x{dp:2d}: {t:8.3f} ms  weights {W/t/1e9:6.0f} GB/s ({W/t/1e9/6545.6:.2f} of HBM)  {fl/t/1e9:7.1f} TF/s", flush=True)
