"""Per-bucket forward roofline on one B200 (evidence for the north_star's two
targets: short buckets >= 60% of HBM roofline, long prefill >= 60% of bf16
tensor peak).

For every CUDA-graph bucket (l_pad, depth) of the reference GraphGrid
(scheduler.hpp:21-32) and for 512-token long-prefill chunks
(scheduler.hpp:46, chunk history H + (k-1)*C_l, scheduler.cpp:332), time the
full-depth forward (lp_submit/lp_wait: CUDA events on the instance stream,
median of N after warm-up) and compare it with the forward's roofline floor
from SURVEY.md §8(d), real (unpadded) tokens:

    bytes = W + 2*V*h + sum (H_i+L_i)*kvB + sum L_i*h*2
    flops = 2*P*sum L + 4*nq*d*layers*sum L*(H+(L+1)/2) + 2*V*h*n_req
    floor = max(bytes / HBM_peak, flops / TC_peak);  frac = floor / t

Members of bucket l_pad draw L ~ U(l_pad/2+1, l_pad) (the bucket's real range,
scheduler.cpp:69-73); `--hist H` gives every member H tokens of resident
history (a re-prefill bucket; the history is prefilled first, untimed).
usage: bucket_roofline.py MODEL [--hist H] [--depths 1,2,..] [--lengths ..] [--long] [--iters N]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402


def peaks():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"] * 1e9, d["bf16_tflops"] * 1e12, d.get("bf16_tflops_sustained", d["bf16_tflops"]) * 1e12
    return 6545.6e9, 1664.4e12, 1402.6e12


def work(m, rows):
    Vh = m.vocab * m.hidden
    b = m.weight_bytes + 2 * Vh + sum((h + l) * m.kv_bytes_per_token for l, h in rows) + \
        sum(l for l, _ in rows) * m.hidden * 2
    f = 2.0 * m.params_nonembed * sum(l for l, _ in rows) + \
        4.0 * m.n_q_heads * m.head_dim * m.layers * sum(l * (h + (l + 1) / 2) for l, h in rows) + 2.0 * Vh * len(rows)
    return b, f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("model")
    ap.add_argument("--hist", type=int, default=0)
    ap.add_argument("--lengths", default="8,16,32,64,128,256")
    ap.add_argument("--depths", default="1,2,4,8,16,32,64")
    ap.add_argument("--long", action="store_true", help="also 512-token chunks at H in {0,512,1536,3584}")
    ap.add_argument("--long-first", action="store_true", help="run the long chunks before the graph buckets")
    ap.add_argument("--long-h", default="0,512,1536,3584", help="histories of the long chunks")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    m = MODELS[a.model]
    lengths = [int(x) for x in a.lengths.split(",") if x]
    depths = [int(x) for x in a.depths.split(",") if x]
    max_tok = max([lp * dp for lp in lengths for dp in depths] + [512])
    max_mem = max(depths)
    hist_tokens = (a.hist + 256) * max_mem * 2 + 8192
    pages = max(1024, hist_tokens // 64 + 256)
    hbm, tc_burst, tc_sus = peaks()
    inst = PrefillInstance(m, max_tokens=max(max_tok, 4096), max_members=max_mem, kv_pages=pages)
    inst.capture_graphs(lengths=lengths, depths=depths)
    rng = np.random.default_rng(0)
    sid = [0]

    def new_members(lp, dp, H):
        ms = []
        for _ in range(dp):
            L = int(rng.integers(lp // 2 + 1, lp + 1)) if lp > 1 else 1
            s = sid[0]
            sid[0] += 1
            done = 0
            while done < H:  # resident history (untimed), eager chunks of <= 4096 tokens
                c = min(4096, H - done)
                inst.forward(c, 1, KIND_STANDARD, [Member(s, s, c, done)],
                             rng.integers(0, m.vocab, c).astype(np.int32))
                done += c
            ms.append(Member(s, s, L, H))
        return ms

    res = []

    def run(lp, dp, kind, H, label):
        ts, rows = [], None
        for it in range(a.iters + 2):
            ms = new_members(lp, dp, H)
            if label == "long":
                ms = [Member(ms[0].req_id, ms[0].session_id, lp, H)]
            toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in ms)).astype(np.int32)
            t = inst.forward(lp, dp, kind, ms, toks)
            if it >= 2:
                ts.append(t)
            rows = [(x.new_tokens, x.history) for x in ms]
            for x in ms:
                inst.release(x.session_id)
        t = float(np.median(ts)) * 1e-3
        b, f = work(m, rows)
        fl_h, fl_t = b / hbm, f / tc_sus
        bound = "hbm" if fl_h > fl_t else "tensor"
        r = {"kind": label, "l_pad": lp, "depth": dp, "H": H, "tokens": sum(l for l, _ in rows), "ms": t * 1e3,
             "bound": bound, "hbm_gbs": b / t / 1e9, "tflops": f / t / 1e12,
             "frac_roofline": max(fl_h, fl_t) / t, "frac_hbm": b / t / hbm, "frac_tensor_sustained": f / t / tc_sus,
             "frac_tensor_burst": f / t / tc_burst}
        res.append(r)
        print(f"{label:5s} {lp:4d}x{dp:2d} H={H:5d} T={r['tokens']:6d} {r['ms']:9.3f} ms  {bound:6s} "
              f"{r['hbm_gbs']:7.0f} GB/s ({r['frac_hbm']:.2f})  {r['tflops']:7.1f} TF/s "
              f"({r['frac_tensor_sustained']:.2f} sus)  roofline {r['frac_roofline']:.2f}", flush=True)

    def longs():
        for H in [int(x) for x in a.long_h.split(",")]:
            run(512, 1, KIND_STANDARD, H, "long")

    if a.long and a.long_first:
        longs()
    for dp in depths:
        for lp in lengths:
            run(lp, dp, KIND_GRAPH, a.hist, "graph")
    if a.long and not a.long_first:
        longs()
    out = {"model": a.model, "hist": a.hist, "peaks": {"hbm_gbs": hbm / 1e9, "tc_burst_tflops": tc_burst / 1e12,
                                                        "tc_sustained_tflops": tc_sus / 1e12}, "buckets": res}
    p = Path(a.out or f"gpurun_out/buckets_{a.model}_h{a.hist}.json")
    p.parent.mkdir(exist_ok=True)
    p.write_text(json.dumps(out, indent=1))
    inst.close()


if __name__ == "__main__":
    main()
