"""Per-projection GEMM timing with the executor's real launch plans."""
import sys
sys.path.insert(0, '.')
from paper_2601_11589_b200.instance import MODELS, PrefillInstance
name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-32b"
m = MODELS[name].with_layers(1)
inst = PrefillInstance(m, max_tokens=8192, max_members=64, kv_pages=64, use_graphs=False)
h, I, d = m.hidden, m.intermediate, m.head_dim
shapes = {0: ((m.n_q_heads + 2 * m.n_kv_heads) * d, h), 1: (h, m.n_q_heads * d), 2: (2 * I, h), 3: (h, I)}
names = {0: "qkv", 1: "o", 2: "gate/up", 3: "down"}
for T in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "16,64,128,256,464,512,1024,2048,4096".split(","))]:
    t_cap = T if T > 256 else {16: 16, 64: 64, 128: 128, 256: 256}.get(T, T)
    line = [f"T={T:5d}"]
    tot_ms = tot_f = tot_b = 0
    for w in range(4):
        M, K = shapes[w]
        ms = inst.time_gemm(0, w, t_cap, T, iters=20)
        fl = 2.0 * M * K * T
        by = M * K * 2
        tot_ms += ms; tot_f += fl; tot_b += by
        line.append(f"{names[w]} {ms*1e3:7.1f}us {fl/ms/1e9:6.0f}TF {by/ms/1e6:5.0f}GB/s")
    line.append(f"| layer {tot_ms*1e3:7.1f}us {tot_f/tot_ms/1e9:5.0f}TF/s {tot_b/tot_ms/1e6:5.0f}GB/s")
    print("  ".join(line), flush=True)
