"""B200 calibration of the reference's closed-form service-time model.

The reference's scheduler reasons with an analytical forward cost
(`batch_service_time`, /root/reference/proj/src/cost_model.cpp:128-148):

    t = kappa_kind + depth^(eta-1) * sum_i [ alpha*l*(l + 2H_i) + beta*l + gamma_w*l + gamma_r*H_i ]

with l = l_pad for BatchShape launches (graph or standard: padding and dummy
rows billed, cost_model.cpp:141) and l = L_i without the depth factor for
packed FCFS batches (cost_model.cpp:150-158), and fits (alpha, beta, gamma_w,
gamma_r) from measured (L, H, t_comp, t_mem) samples with a clamped 2-column
least squares (`fit_params`, cost_model.cpp:63-120; "fitting
at runtime"). A real forward does not expose t_comp and t_mem separately, so
this module fits the whole service-time model to measured B200 forwards:

  * for a fixed eta the model is linear in (kappa_graph, kappa_std, alpha,
    beta + gamma_w, gamma_r): non-negative least squares on relative error;
  * eta by a 1-D search over (0.3, 1];
  * beta + gamma_w is split with the roofline: beta = the per-token tensor
    time 2*P / TC_sustained (the compute part of t_comp = alpha*L(L+2H) +
    beta*L), gamma_w = the remainder (per-token memory traffic).

The result is a set of reference config keys (cost.*, exec.*) that make the
reference's own engine (and this repo's byte-identical one) predict B200
service times. Host-side only: numpy + scipy.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.optimize import nnls


@dataclass
class Sample:
    """One measured forward: shape + members (L_i, H_i) + device ms."""
    l_pad: int
    depth: int
    kind: str      # "graph" | "standard" (BatchShape kinds) | "packed" (FCFS)
    members: list  # [(L, H), ...] real members (dummy rows are implied by depth)
    ms: float


@dataclass
class Calibration:
    alpha: float
    beta: float
    gamma_w: float
    gamma_r: float
    kappa_graph_ms: float
    kappa_std_ms: float
    eta: float
    rel_rmse: float
    max_rel_err: float

    def config(self) -> dict:
        """Reference config keys (config.cpp:211-229)."""
        return {"cost.alpha": f"{self.alpha:.6e}", "cost.beta": f"{self.beta:.6e}",
                "cost.gamma_w": f"{self.gamma_w:.6e}", "cost.gamma_r": f"{self.gamma_r:.6e}",
                "exec.kappa_graph_ms": f"{self.kappa_graph_ms:.6f}", "exec.kappa_std_ms": f"{self.kappa_std_ms:.6f}",
                "exec.eta": f"{self.eta:.4f}"}

    def predict(self, s: Sample) -> float:
        return predict(s, self.alpha, self.beta + self.gamma_w, self.gamma_r, self.kappa_graph_ms,
                       self.kappa_std_ms, self.eta)

    def prefill_boundary(self) -> float:
        """L where t_comp = t_mem for H = 0 (cost_model.cpp:43-46)."""
        return max(0.0, (self.gamma_w - self.beta) / self.alpha)


def _rows(s: Sample):
    """Billed rows (cost_model.cpp:128-158): a BatchShape bills every member
    and every dummy row (sim.cpp:249-253: L = 0, H = 0) at l_pad; a packed
    batch bills the real members only."""
    if s.kind == "packed":
        return list(s.members)
    rows = [(s.l_pad, h) for (_, h) in s.members]
    return rows + [(s.l_pad, 0)] * (s.depth - len(s.members))


def _design(s: Sample, eta: float) -> np.ndarray:
    rows = _rows(s)
    f = s.depth ** (eta - 1.0) if s.kind != "packed" else 1.0
    a = sum(l * (l + 2.0 * h) for l, h in rows) * f
    b = sum(l for l, _ in rows) * f
    r = sum(h for _, h in rows) * f
    g = s.kind == "graph"
    return np.array([1.0 if g else 0.0, 0.0 if g else 1.0, a, b, r])


def predict(s: Sample, alpha, b_tok, gamma_r, kg, ks, eta) -> float:
    return float(_design(s, eta) @ np.array([kg, ks, alpha, b_tok, gamma_r]))


def _fit_fixed_eta(samples, eta):
    X = np.stack([_design(s, eta) for s in samples])
    y = np.array([s.ms for s in samples])
    w = 1.0 / y  # relative error
    coef, _ = nnls(X * w[:, None], y * w)
    pred = X @ coef
    rel = (pred - y) / y
    return coef, float(np.sqrt(np.mean(rel ** 2))), float(np.max(np.abs(rel)))


def fit(samples: list[Sample], beta_compute: float, etas=None) -> Calibration:
    """Fit the service-time model. beta_compute: per-token tensor time in ms
    (2 * non-embedding params / sustained bf16 FLOP/s)."""
    if len(samples) < 6:
        raise ValueError("need >= 6 samples")
    etas = np.linspace(0.3, 1.0, 71) if etas is None else etas
    best = None
    for eta in etas:
        coef, rmse, mx = _fit_fixed_eta(samples, float(eta))
        if best is None or rmse < best[1]:
            best = (coef, rmse, mx, float(eta))
    coef, rmse, mx, eta = best
    kg, ks, alpha, b_tok, gamma_r = (float(c) for c in coef)
    alpha = max(alpha, 1e-12)  # the reference requires alpha > 0 (cost_model.cpp:9-13)
    beta = min(beta_compute, b_tok)
    return Calibration(alpha=alpha, beta=beta, gamma_w=b_tok - beta, gamma_r=gamma_r, kappa_graph_ms=kg,
                       kappa_std_ms=max(ks, kg), eta=eta, rel_rmse=rmse, max_rel_err=mx)
