"""Cost-model calibration (paper_2601_11589_b200/calibrate.py): recovers the
reference service-time model's parameters from synthetic samples generated
by that model (the analogue of the reference's fit-recovery acceptance
criterion c4, acceptance.cpp), and the fitted keys drive the engine."""
import numpy as np

from paper_2601_11589_b200 import calibrate as C
from paper_2601_11589_b200 import engine as E
from paper_2601_11589_b200 import scenarios as S


def _samples(true, rng):
    out = []
    for lp in (16, 64, 128, 256):
        for dp in (1, 2, 4, 8):
            for H in (0, 1024):
                ms = [(int(rng.integers(lp // 2 + 1, lp + 1)), H) for _ in range(dp)]
                s = C.Sample(lp, dp, "graph", ms, 0.0)
                s.ms = C.predict(s, *true)
                out.append(s)
    for L, H in ((512, 0), (512, 512), (512, 1536), (300, 3584), (256, 0)):
        s = C.Sample(L, 1, "standard", [(L, H)], 0.0)
        s.ms = C.predict(s, *true)
        out.append(s)
    return out


def test_fit_recovers_reference_model():
    rng = np.random.default_rng(0)
    true = (2e-5, 0.015, 0.002, 0.05, 0.5, 0.7)  # alpha, beta+gamma_w, gamma_r, kappa_g, kappa_std, eta
    cal = C.fit(_samples(true, rng), beta_compute=0.005)
    assert abs(cal.eta - 0.7) < 1e-9
    assert abs(cal.alpha / 2e-5 - 1) < 1e-6 and abs(cal.gamma_r / 0.002 - 1) < 1e-6
    assert abs((cal.beta + cal.gamma_w) / 0.015 - 1) < 1e-6 and abs(cal.beta - 0.005) < 1e-12
    assert abs(cal.kappa_graph_ms - 0.05) < 1e-9 and abs(cal.kappa_std_ms - 0.5) < 1e-9
    assert cal.rel_rmse < 1e-9


def test_calibrated_keys_drive_the_engine(tmp_path):
    cal = C.Calibration(alpha=3e-6, beta=0.004, gamma_w=0.006, gamma_r=0.0005, kappa_graph_ms=2.6,
                        kappa_std_ms=2.9, eta=0.9, rel_rmse=0.0, max_rel_err=0.0)
    cfg = S.text(S.merged(S.SHORT_7B, sim__duration_ms=3000, **{k.replace(".", "__"): v for k, v in cal.config().items()}))
    st = E.simulate(cfg, "", tmp_path)
    assert st.completed > 0 and st.ttft_p50_ms > 2.6
