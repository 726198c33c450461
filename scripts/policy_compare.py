"""The paper's system-level comparison on real B200 forwards: LAPS
(dual queues + AWD batching + length-bucket graphs, temporal
disaggregation on one instance) vs the reference's two baselines,
FCFS-unified packed batching and bucketing without disaggregation
(sim.cpp:379-411 policies) — plus LAPS with deadline-free admission
(token_max batching, scheduler.cpp:288-320) — all in LIVE mode — the engine clock advances by
the measured GPU time of every dispatched forward, so TTFT and SLO
violations are what this B200 path delivers under each policy.

Workload: Qwen2.5-7B-shaped, the mixed multi-turn stream of BASELINE.json
config 3 (short 16-255 / long 1500-2600, later turns mostly short
re-prefills over the session's KV), one GPU, several offered loads.
Writes gpurun_out/policy_compare.json.
usage: policy_compare.py [duration_ms] [loads...]"""
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200 import engine as E  # noqa: E402
from paper_2601_11589_b200 import scenarios as S  # noqa: E402
from paper_2601_11589_b200.instance import QWEN25_7B, PrefillInstance  # noqa: E402

dur = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
loads = [float(x) for x in sys.argv[2:]] or [0.01, 0.02, 0.03]
inst = PrefillInstance(QWEN25_7B, max_tokens=16384, max_members=64)
inst.capture_graphs()
POLICIES = {
    "laps": {"sim.policy": "laps", "sim.disagg": "temporal"},
    "laps_deadline_free": {"sim.policy": "laps", "sim.disagg": "temporal", "sched.mode": "deadline_free"},
    "bucket_no_disagg": {"sim.policy": "bucket_no_disagg"},
    "fcfs_unified": {"sim.policy": "fcfs_unified"},
    # B200-tuned LAPS: one forward per long prompt up to 2048 tokens (C_l = 2048) so a
    # long prompt pays the weight stream once instead of once per 512-token chunk.
    "laps_cl2048": {"sim.policy": "laps", "sim.disagg": "temporal", "sched.c_l_tokens": "2048"},
    "laps_deadline_free_cl2048": {"sim.policy": "laps", "sim.disagg": "temporal", "sched.mode": "deadline_free",
                                  "sched.c_l_tokens": "2048"},
}

out = {"model": "qwen2.5-7b", "duration_ms": dur, "runs": []}
for lam in loads:
    for name, pol in POLICIES.items():
        cfg = S.merged(S.REPREFILL_7B, sim__duration_ms=dur, workload__lambda_per_ms=lam,
                       **{k.replace(".", "__"): v for k, v in pol.items()})
        d = Path(tempfile.mkdtemp(prefix=f"pol_{name}_"))
        st = E.simulate(S.text(cfg), "", d, mode=E.LIVE, instances=[inst], token_seed=7)
        m = json.loads((d / "metrics.json").read_text())
        row = {"policy": name, "lambda_per_ms": lam, "gpu_forwards": st.gpu_forwards, "gpu_ms_total": st.gpu_ms_total,
               **{f"{cls}_{k}": m[cls][k] for cls in ("overall", "short", "long")
                  for k in ("completed", "ttft_p50_ms", "ttft_p90_ms", "ttft_p99_ms", "slo_violation")}}
        out["runs"].append(row)
        print(f"lambda={lam:.3f} {name:17s} TTFT p50/p90 all {row['overall_ttft_p50_ms']:8.1f}/{row['overall_ttft_p90_ms']:8.1f} "
              f"short {row['short_ttft_p50_ms']:8.1f}/{row['short_ttft_p90_ms']:8.1f} ms  SLO viol {row['overall_slo_violation']:.3f}  "
              f"completed {row['overall_completed']}", flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/policy_compare.json").write_text(json.dumps(out, indent=1))
inst.close()
