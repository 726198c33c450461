"""Profile one forward of a given shape: W eager-free warmups then replays.
usage: prof_forward.py LPAD DEPTH [layers] [model]
Launch accounting for ncu: capture_graphs runs 1 eager warm-up forward; each
forward = 1 + layers*9 + 3 kernel launches."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_11589_b200.instance import MODELS, Member, PrefillInstance, KIND_GRAPH, KIND_STANDARD
lp, dp = int(sys.argv[1]), int(sys.argv[2])
model = MODELS[sys.argv[4] if len(sys.argv) > 4 else "qwen2.5-7b"]
if len(sys.argv) > 3 and int(sys.argv[3]) > 0:
    model = model.with_layers(int(sys.argv[3]))
inst = PrefillInstance(model, max_tokens=max(lp * dp, 512), max_members=max(dp, 16), kv_pages=2048)
graph = lp <= 256
if graph:
    inst.capture_graphs(lengths=(lp,), depths=(dp,))
rng = np.random.default_rng(0)
ts = []
for it in range(8):
    ms = [Member(i, 1000 * it + i, lp if lp <= 16 else int(rng.integers(lp // 2 + 1, lp + 1)), 0) for i in range(dp)]
    toks = rng.integers(0, model.vocab, sum(m.new_tokens for m in ms)).astype(np.int32)
    ts.append(inst.forward(lp, dp, KIND_GRAPH if graph else KIND_STANDARD, ms, toks))
    for m in ms: inst.release(m.session_id)
print(f"shape {lp}x{dp} layers {model.layers}: median {np.median(ts[2:]):.3f} ms  all {np.round(ts, 3).tolist()}")
