import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import forward_oracle as FO
from paper_2601_11589_b200.instance import QWEN25_7B, Member, PrefillInstance, KIND_GRAPH, KIND_STANDARD
cfg = QWEN25_7B.with_layers(2)
inst = PrefillInstance(cfg, max_tokens=2048, max_members=16, kv_pages=64)
inst.capture_graphs(lengths=(256,), depths=(2, 8))
ms = [Member(0, 0, 200, 0), Member(1, 1, 77, 0)]
toks = np.concatenate([FO.tokens(7, m.session_id, m.history, m.new_tokens, cfg.vocab) for m in ms])
res = {}
for name, (lp, dp, kind) in {"g256x2": (256, 2, KIND_GRAPH), "g256x8": (256, 8, KIND_GRAPH), "eager": (256, 2, KIND_STANDARD)}.items():
    inst.forward(lp, dp, kind, ms, toks)
    res[name] = torch.from_numpy(inst.logits())
o = FO.OracleModel(FO.with_layers(FO.QWEN25_7B, 2))
res["oracle"] = o.forward([(m.session_id, m.new_tokens, m.history) for m in ms],
                          [FO.tokens(7, m.session_id, m.history, m.new_tokens, cfg.vocab) for m in ms])
names = list(res)
for i in range(len(names)):
    for j in range(i + 1, len(names)):
        d = (res[names[i]] - res[names[j]]).abs()
        print(f"{names[i]:>7} vs {names[j]:<7} max {d.max().item():.4f} mean {d.mean().item():.5f}")
