import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import forward_oracle as FO
from paper_2601_11589_b200.instance import QWEN25_7B, Member, PrefillInstance, KIND_GRAPH
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = QWEN25_7B.with_layers(L)
inst = PrefillInstance(cfg, max_tokens=1024, max_members=16, kv_pages=64)
inst.capture_graphs(lengths=(256,), depths=(2,))
o = FO.OracleModel(FO.with_layers(FO.QWEN25_7B, L))
ms = [Member(0, 0, 200, 0), Member(1, 1, 77, 0)]
toks = [FO.tokens(7, m.session_id, m.history, m.new_tokens, cfg.vocab) for m in ms]
inst.forward(256, 2, KIND_GRAPH, ms, np.concatenate(toks))
want = o.forward([(m.session_id, m.new_tokens, m.history) for m in ms], toks)
got = torch.from_numpy(inst.logits())
d = (got - want).abs()
print("logits: max", d.max().item(), "mean", d.mean().item(), "std(want)", want.std().item(),
      "cos", torch.nn.functional.cosine_similarity(got, want, dim=1).tolist())
for l in range(L):
    k, v = inst.read_kv(0, l, 0, 200)
    kk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).float()
    vv = torch.from_numpy(v.view(np.int16)).view(torch.bfloat16).float()
    K, V = o.read_kv(0, l, 0, 200)
    print(f"layer {l}: K max {(kk-K).abs().max().item():.4g} mean {(kk-K).abs().mean().item():.3g} |K| {K.abs().mean().item():.3g};"
          f" V max {(vv-V).abs().max().item():.4g} mean {(vv-V).abs().mean().item():.3g} |V| {V.abs().mean().item():.3g}")
    # fraction of exactly-equal bf16 values
    print("   K exact frac", (kk == K).float().mean().item(), " V exact frac", (vv == V).float().mean().item())
