"""Per-projection GEMM time vs live tokens through the instance's own launch
plan (split-K, tile width, CTA pairs), CUDA events, Qwen2.5-7B/32B shapes.
usage: gemm_table.py [model] [t_caps...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import MODELS, PrefillInstance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
m = MODELS[name]
caps = [int(x) for x in sys.argv[2:]] or [16, 64, 128, 256, 384, 512, 768, 1024, 2048, 4096]
inst = PrefillInstance(m.with_layers(1), max_tokens=max(caps), max_members=64, kv_pages=64)
h, I, D = m.hidden, m.intermediate, m.head_dim
shapes = {0: ("qkv", (m.n_q_heads + 2 * m.n_kv_heads) * D, h), 1: ("o", h, m.n_q_heads * D),
          2: ("gate/up", 2 * I, h), 3: ("down", h, I)}
HBM, TC = 6545.6e9, 1664.4e12
tot = {}
for t in caps:
    row = []
    for w, (nm, M, K) in shapes.items():
        ms = inst.time_gemm(0, w, t, t, iters=20)
        b = M * K * 2 + t * K * 2
        f = 2.0 * M * K * t
        floor = max(b / HBM, f / TC)
        row.append(f"{nm}:{ms * 1e3:7.1f}us {floor / (ms * 1e-3):4.2f}")
        tot[t] = tot.get(t, [0, 0])
        tot[t][0] += ms * 1e-3
        tot[t][1] += floor
    print(f"T={t:5d} " + "  ".join(row) + f"  | layer GEMMs {tot[t][0] * 1e6:7.1f}us frac {tot[t][1] / tot[t][0]:.2f}",
          flush=True)
