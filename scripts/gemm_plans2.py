"""Per-projection GEMM timing at (t_cap, n_live) with the executor's plans and realistic inputs."""
import sys
sys.path.insert(0, '.')
from paper_2601_11589_b200.instance import MODELS, PrefillInstance
name = sys.argv[1]
m = MODELS[name].with_layers(1)
inst = PrefillInstance(m, max_tokens=16384, max_members=64, kv_pages=64, use_graphs=False)
h, I, d = m.hidden, m.intermediate, m.head_dim
shapes = {0: ((m.n_q_heads + 2 * m.n_kv_heads) * d, h), 1: (h, m.n_q_heads * d), 2: (2 * I, h), 3: (h, I)}
names = {0: "qkv", 1: "o", 2: "gate/up", 3: "down"}
for pair in sys.argv[2:]:
    t_cap, n_live = map(int, pair.split(":"))
    line = [f"t_cap={t_cap:5d} live={n_live:5d}"]
    tot_ms = tot_f = 0
    for w in range(4):
        M, K = shapes[w]
        ms = inst.time_gemm(0, w, t_cap, n_live, iters=20)
        fl = 2.0 * M * K * n_live
        tot_ms += ms; tot_f += fl
        line.append(f"{names[w]} {ms*1e3:7.1f}us {fl/ms/1e9:5.0f}TF")
    line.append(f"| layer {tot_ms*1e3:7.1f}us {tot_f/tot_ms/1e9:5.0f}TF/s")
    print("  ".join(line), flush=True)
inst.close()
