"""Launch the bench's dominant kernel (gate/up GEMM + fused SiLU*up of one
decoder layer) at a given step capacity / live token count through the
instance's own launch plan, for `ncu --set full` (profiles/*_dominant_kernel.json).
usage: prof_dominant.py T_CAP N_LIVE [ITERS] [WHICH: 0 qkv, 1 o, 2 gate/up, 3 down] [MODEL]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import MODELS, PrefillInstance  # noqa: E402

t_cap, n_live = int(sys.argv[1]), int(sys.argv[2])
which = int(sys.argv[4]) if len(sys.argv) > 4 else 2
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
model = MODELS[sys.argv[5] if len(sys.argv) > 5 else "qwen2.5-7b"]
inst = PrefillInstance(model.with_layers(1), max_tokens=max(t_cap, 512), max_members=64, kv_pages=64)
ms = inst.time_gemm(0, which, t_cap, n_live, iters=iters)
print(f"gemm {which} t_cap={t_cap} n_live={n_live}: {ms * 1e3:.1f} us")
