"""BASELINE.json configs 1-4 on one B200 (evidence for profiles/; not the driver's bench line).

For each config: a REPLAY run (reference cost-model clock -> batch composition
byte-identical to the reference scheduler; every dispatch executes on the GPU,
multi-turn history stays resident / is filled, long prompts run as 512-token
chunks) reports GPU-time throughput and forward-level roofline numbers; a LIVE
run (clock = measured forward times) reports TTFT p50/p90.
usage: run_configs.py [c1 c2 c3 c4]
"""
import csv
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200 import engine as E  # noqa: E402
from paper_2601_11589_b200 import scenarios as S  # noqa: E402
from paper_2601_11589_b200.instance import MODELS, PrefillInstance  # noqa: E402

def _peaks():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"] * 1e9, d["bf16_tflops"] * 1e12, d.get("bf16_tflops_sustained", d["bf16_tflops"]) * 1e12
    return 6545.6e9, 1664.4e12, 1402.6e12


PEAK_HBM, PEAK_TC, PEAK_TC_SUS = _peaks()

CONFIGS = {
    "c1": ("tiny", S.DEFAULT, {}),
    "c2": ("qwen2.5-7b", S.SHORT_7B, {"workload.lambda_per_ms": "0.3", "sim.duration_ms": "10000"}),
    "c3": ("qwen2.5-7b", S.REPREFILL_7B, {"sim.duration_ms": "30000"}),
    "c4": ("qwen2.5-32b", S.LMSYS_32B, {"sim.duration_ms": "15000"}),
}


def work_of(model, trace, events):
    """Algorithmic bytes / flops of every dispatched forward."""
    by = {r.id: r for r in trace}
    W = model.weight_bytes
    Vh = model.vocab * model.hidden
    kvB = model.kv_bytes_per_token
    P = model.params_nonembed
    byts = flops = 0.0
    chunk_done = {}
    for line in events.read_text().splitlines():
        r = json.loads(line)
        if r["kind"] != "dispatch":
            continue
        rows = []
        for rid in r["reqs"]:
            t = by[rid]
            if r["chunk"]:
                done = chunk_done.get(rid, 0)
                rows.append((r["real"], t.H + done))
                chunk_done[rid] = done + r["real"]
            else:
                rows.append((t.L, t.H))
        byts += W + 2 * Vh + sum((h + l) * kvB for l, h in rows) + sum(l for l, _ in rows) * model.hidden * 2
        flops += (2.0 * P * sum(l for l, _ in rows) + 4.0 * model.n_q_heads * model.head_dim * model.layers *
                  sum(l * (h + (l + 1) / 2) for l, h in rows) + 2.0 * Vh * len(rows))
    return byts, flops


def main(names):
    out = {}
    for name in names:
        mname, base, over = CONFIGS[name]
        model = MODELS[mname]
        cfg = S.text({**base, **over})
        t0 = time.time()
        inst = PrefillInstance(model, max_tokens=16384, max_members=64)
        inst.capture_graphs()
        setup = time.time() - t0
        d = Path(tempfile.mkdtemp(prefix=f"cfg_{name}_"))
        st = E.simulate(cfg, "", d / "replay", mode=E.REPLAY, instances=[inst], token_seed=7)
        E.dump_trace(cfg, "", d / "trace.txt")
        trace = E.load_trace_dump(d / "trace.txt")
        byts, flops = work_of(model, trace, d / "replay" / "events.log")
        gpu_s = st.gpu_ms_total / 1000.0
        live = E.simulate(cfg, "", d / "live", mode=E.LIVE, instances=[inst], token_seed=7)
        rows = list(csv.DictReader(open(d / "replay" / "forwards.csv")))
        # Per-forward roofline: floor_i = max(bytes_i / HBM, flops_i / sustained bf16) from each
        # dispatch's real tokens / histories; frac = sum floor / sum measured.
        Vh = model.vocab * model.hidden
        fl = {"graph": [0.0, 0.0], "standard": [0.0, 0.0], "all": [0.0, 0.0]}
        for rw in rows:
            T, Hs, pairs, n = int(rw["tokens"]), int(rw["hist_tokens"]), float(rw["attn_pairs"]), int(rw["members"])
            b = model.weight_bytes + 2 * Vh + (T + Hs) * model.kv_bytes_per_token + T * model.hidden * 2
            f = 2.0 * model.params_nonembed * T + 4.0 * model.n_q_heads * model.head_dim * model.layers * pairs + 2.0 * Vh * n
            floor = max(b / PEAK_HBM, f / PEAK_TC_SUS)
            t = float(rw["gpu_ms"]) * 1e-3
            for k in ("graph" if rw["graph"] == "1" else "standard", "all"):
                fl[k][0] += floor
                fl[k][1] += t
        out[name] = {
            "model": mname, "requests": st.arrivals, "dispatches": st.dispatches, "gpu_forwards": st.gpu_forwards,
            "history_fills": st.fill_forwards, "gpu_seconds": gpu_s,
            "gpu_req_per_s": st.completed / gpu_s, "forward_hbm_tb_s": byts / gpu_s / 1e12,
            "forward_tflops": flops / gpu_s / 1e12, "frac_hbm": byts / gpu_s / PEAK_HBM,
            "frac_tensor": flops / gpu_s / PEAK_TC,
            "live": {"ttft_p50_ms": live.ttft_p50_ms, "ttft_p90_ms": live.ttft_p90_ms, "rps": live.rps,
                     "slo_violation": live.slo_violation},
            "replay_cost_model": {"ttft_p50_ms": st.ttft_p50_ms, "ttft_p90_ms": st.ttft_p90_ms},
            "graph_forwards": sum(1 for r in rows if r["graph"] == "1"), "setup_s": setup,
            "frac_roofline": {k: (v[0] / v[1] if v[1] else None) for k, v in fl.items()},
        }
        print(name, json.dumps(out[name]), flush=True)
        inst.close()
    return out


if __name__ == "__main__":
    res = main(sys.argv[1:] or list(CONFIGS))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/configs.json").write_text(json.dumps(res, indent=1))
