"""Full-depth parity spot check (SURVEY.md §7 hard part 7: "parity at full
width with reduced depth, spot-check full depth on the box"): Qwen2.5-7B-
shaped, all 28 layers, GPU forward vs the CPU oracle (fp32, all host
threads) on a graph bucket and a re-prefill over the cached pages.
Prints logits max-abs / mean-abs / min cosine and greedy-token agreement.
usage: full_depth_parity.py [layers]"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import forward_oracle as FO  # noqa: E402
from paper_2601_11589_b200.instance import KIND_GRAPH, QWEN25_7B, Member, PrefillInstance  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 28
cfg = QWEN25_7B.with_layers(layers)
t0 = time.time()
oracle = FO.OracleModel(FO.with_layers(FO.QWEN25_7B, layers), threads=os.cpu_count())
print(f"oracle weights {time.time() - t0:.1f}s", flush=True)
inst = PrefillInstance(cfg, max_tokens=1024, max_members=8, kv_pages=64)
inst.capture_graphs(lengths=(64,), depths=(2,))
out = {"layers": layers, "cases": []}
for members in ([Member(0, 0, 40, 0), Member(1, 1, 24, 0)], [Member(2, 0, 30, 40)]):
    toks = [FO.tokens(7, m.session_id, m.history, m.new_tokens, cfg.vocab) for m in members]
    inst.forward(64, 2, KIND_GRAPH, members, np.concatenate(toks))
    t0 = time.time()
    want = oracle.forward([(m.session_id, m.new_tokens, m.history) for m in members], toks)
    got = torch.from_numpy(inst.logits())
    d = (got - want).abs()
    cos = torch.nn.functional.cosine_similarity(got, want, dim=1).min().item()
    nt = inst.next_tokens()
    top2 = torch.topk(want, 2, dim=1).values
    agree = [int(nt[i]) == int(torch.argmax(want[i])) for i in range(len(members))]
    margin = [(top2[i, 0] - top2[i, 1]).item() for i in range(len(members))]
    case = {"members": [(m.new_tokens, m.history) for m in members], "max_abs": d.max().item(),
            "mean_abs": d.mean().item(), "min_cos": cos, "logit_std": want.std().item(),
            "greedy_agree": agree, "top2_margin": margin, "oracle_s": time.time() - t0}
    out["cases"].append(case)
    print(json.dumps(case), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/full_depth_parity_{layers}.json").write_text(json.dumps(out, indent=1))
