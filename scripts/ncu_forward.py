"""One full-depth forward of a given bucket inside an NVTX range "target",
for ncu counter capture (north_star: achieved HBM GB/s for short / re-prefill
buckets, tensor-pipe utilisation for long prefills):

  ncu --nvtx --nvtx-include target/ --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv --log-file X.csv \
      python scripts/ncu_forward.py MODEL KIND L_PAD DEPTH H

KIND graph|standard; members draw L ~ U(l_pad/2+1, l_pad) (graph) or L = l_pad
(standard), each with H tokens of resident history."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

name, kind, lp, dp, H = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
m = MODELS[name]
graph = kind == "graph"
inst = PrefillInstance(m, max_tokens=max(4096, lp * dp), max_members=max(dp, 8), kv_pages=max(512, dp * (H + lp) // 64 + 64))
if graph:
    inst.capture_graphs(lengths=(lp,), depths=(dp,))
rng = np.random.default_rng(0)
sid = [0]


def members():
    out = []
    for _ in range(dp):
        s = sid[0]
        sid[0] += 1
        done = 0
        while done < H:
            c = min(4096, H - done)
            inst.forward(c, 1, KIND_STANDARD, [Member(s, s, c, done)], rng.integers(0, m.vocab, c).astype(np.int32))
            done += c
        L = int(rng.integers(lp // 2 + 1, lp + 1)) if graph and lp > 8 else lp
        out.append(Member(s, s, L, H))
    return out


for it in range(3):
    ms = members()
    toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in ms)).astype(np.int32)
    if it == 2:
        torch.cuda.nvtx.range_push("target")
    t = inst.forward(lp, dp, KIND_GRAPH if graph else KIND_STANDARD, ms, toks)
    if it == 2:
        torch.cuda.nvtx.range_pop()
        print(f"{name} {kind} {lp}x{dp} H={H} tokens={sum(x.new_tokens for x in ms)}: {t:.3f} ms (event-timed)")
    for x in ms:
        inst.release(x.session_id)
