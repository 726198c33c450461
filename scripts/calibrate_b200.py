"""Calibrate the reference's service-time model to B200 forwards and check
what the calibrated reference engine predicts against the live GPU engine.

1. Measure full-depth Qwen2.5-7B forwards (CUDA events): graph buckets
   l_pad x depth at H = 0 and H = 1024, and standard long-prefill chunks.
2. Fit (alpha, beta, gamma_w, gamma_r, kappa_graph, kappa_std, eta) with
   paper_2601_11589_b200.calibrate.fit.
3. Run config 2 (short-only stream) at 0.25 req/ms through the engine three
   ways: LIVE on the GPU (clock = measured forwards), and the cost-model
   engine with the reference's default parameters and with the calibrated
   ones; report TTFT p50/p90 and service-time error.
Writes gpurun_out/calibration.json.
"""
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200 import calibrate as C  # noqa: E402
from paper_2601_11589_b200 import engine as E  # noqa: E402
from paper_2601_11589_b200 import scenarios as S  # noqa: E402
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, QWEN25_7B, Member, PrefillInstance  # noqa: E402

m = QWEN25_7B
inst = PrefillInstance(m, max_tokens=16384, max_members=64, kv_pages=8192)
inst.capture_graphs()
rng = np.random.default_rng(3)
sid = [0]


def member(L, H):
    s = sid[0]
    sid[0] += 1
    done = 0
    while done < H:
        c = min(4096, H - done)
        inst.forward(c, 1, KIND_STANDARD, [Member(s, s, c, done)], rng.integers(0, m.vocab, c).astype(np.int32))
        done += c
    return Member(s, s, L, H)


def measure(l_pad, depth, kind, rows, reps=3):
    ts = []
    for _ in range(reps + 1):
        ms = [member(L, H) for L, H in rows]
        toks = rng.integers(0, m.vocab, sum(L for L, _ in rows)).astype(np.int32)
        ts.append(inst.forward(l_pad, depth, kind, ms, toks))
        for x in ms:
            inst.release(x.session_id)
    return float(np.median(ts[1:]))


samples = []
for H in (0, 1024):
    for dp in (1, 2, 4, 8, 16):
        for lp in (8, 16, 32, 64, 128, 256):
            if H and dp > 8:
                continue
            n = dp if dp == 1 else max(1, dp - int(rng.integers(0, dp // 2 + 1)))  # some dummy rows
            rows = [(int(rng.integers(lp // 2 + 1, lp + 1)) if lp > 8 else lp, H) for _ in range(n)]
            samples.append(C.Sample(lp, dp, "graph", rows, measure(lp, dp, KIND_GRAPH, rows)))
for L, H in ((512, 0), (512, 512), (512, 1536), (512, 3584), (300, 0), (300, 2048)):
    samples.append(C.Sample(L, 1, "standard", [(L, H)], measure(L, 1, KIND_STANDARD, [(L, H)])))
print(f"{len(samples)} samples", flush=True)

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
beta_compute = 2.0 * m.params_nonembed / (peaks["bf16_tflops_sustained"] * 1e12) * 1e3  # ms per token
cal = C.fit(samples, beta_compute)
print("calibration", cal, flush=True)

# Validation on config 2 at sub-saturation load.
base = S.merged(S.SHORT_7B, workload__lambda_per_ms=0.25, sim__duration_ms=4000)
d = Path(tempfile.mkdtemp(prefix="calib_"))
live = E.simulate(S.text(base), "", d / "live", mode=E.LIVE, instances=[inst], token_seed=7)
ref_default = E.simulate(S.text(base), "", d / "ref")
cal_cfg = S.merged(base, **{k.replace(".", "__"): v for k, v in cal.config().items()})
calibrated = E.simulate(S.text(cal_cfg), "", d / "cal")


def stats(st):
    return {"ttft_p50_ms": st.ttft_p50_ms, "ttft_p90_ms": st.ttft_p90_ms, "rps": st.rps, "dispatches": st.dispatches}


res = {"model": "qwen2.5-7b", "samples": [{"l_pad": s.l_pad, "depth": s.depth, "kind": s.kind, "members": s.members,
                                           "ms": s.ms, "pred_ms": cal.predict(s)} for s in samples],
       "calibration": {**cal.__dict__, "config": cal.config(), "beta_compute_ms_per_token": beta_compute,
                       "prefill_boundary_tokens": cal.prefill_boundary()},
       "validation_c2_lambda0.25": {"live_gpu": stats(live), "cost_model_reference_defaults": stats(ref_default),
                                    "cost_model_calibrated": stats(calibrated)}}
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/calibration.json").write_text(json.dumps(res, indent=1))
print(json.dumps(res["validation_c2_lambda0.25"], indent=1))
print("fit rel rmse", cal.rel_rmse, "max", cal.max_rel_err)
