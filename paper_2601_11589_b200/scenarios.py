"""Scenario definitions (reference config-key vocabulary, config.cpp:159-335).

`DEFAULT` and `MIXED_DRIFT` restate the settings of the reference's two
shipped scenarios (/root/reference/proj/configs/default.cfg:7-61 and
mixed_drift.cfg:7-36) as key/value maps, so nothing here reads the reference
tree at run time. `BASELINE_CONFIGS` are the five BASELINE.json configs.
"""
from __future__ import annotations

DEFAULT = {
    "sim.policy": "laps", "sim.disagg": "spatial", "sim.instances": "4", "sim.controller": "true",
    "sim.initial_short_instances": "1", "sim.duration_ms": "60000", "sim.slo_ms": "400", "sim.seed": "1",
    "workload.lambda_per_ms": "0.03", "workload.short_fraction": "0.63", "workload.short_lo": "16",
    "workload.short_hi": "255", "workload.long_lo": "1024", "workload.long_hi": "2048",
    "workload.turns_lo": "1", "workload.turns_hi": "4", "workload.slo_offset_ms": "400", "workload.seed": "1",
    "cost.alpha": "2e-5", "cost.beta": "0.005", "cost.gamma_w": "0.01012", "cost.gamma_r": "0.002",
    "exec.kappa_graph_ms": "0.05", "exec.kappa_std_ms": "0.5", "exec.eta": "0.7",
    "sched.mode": "sla", "sched.w_min_ms": "1", "sched.w_max_ms": "50", "sched.c_l_tokens": "512",
    "sched.l_m_first": "256", "grid.model_preset": "7b", "grid.mem_budget_mb": "4096",
    "ctrl.dt_ms": "100", "ctrl.t_cool_ms": "1500", "ctrl.tau_hyst": "0.25", "ctrl.n_min": "1", "ctrl.w_u": "0",
}

MIXED_DRIFT = {
    "sim.policy": "laps", "sim.disagg": "spatial", "sim.instances": "8", "sim.controller": "true",
    "sim.initial_short_instances": "4", "sim.duration_ms": "120000", "sim.slo_ms": "400", "sim.seed": "42",
    "workload.lambda_per_ms": "0.08", "workload.short_fraction": "0.63", "workload.short_fraction_later": "0.81",
    "workload.short_lo": "16", "workload.short_hi": "255", "workload.long_lo": "1500", "workload.long_hi": "2600",
    "workload.turns_lo": "2", "workload.turns_hi": "6", "workload.slo_offset_ms": "400", "workload.seed": "42",
    "grid.model_preset": "7b", "grid.mem_budget_mb": "4096",
    "ctrl.n_min": "1", "ctrl.t_cool_ms": "2000", "ctrl.tau_hyst": "0.5", "ctrl.w_u": "0",
}


def text(cfg: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in cfg.items())


def merged(base: dict, **over) -> dict:
    out = dict(base)
    for k, v in over.items():
        out[k.replace("__", ".")] = str(v)
    return out


# BASELINE.json configs.
SHORT_7B = {  # config 2: Qwen2.5-7B, short-only (<256) with waiting window, 1 GPU temporal
    "sim.policy": "laps", "sim.disagg": "temporal", "sim.instances": "1", "sim.duration_ms": "20000",
    "sim.slo_ms": "400", "workload.lambda_per_ms": "0.5", "workload.short_fraction": "1.0",
    "workload.short_fraction_later": "1.0", "workload.short_lo": "8", "workload.short_hi": "255",
    "workload.turns_lo": "1", "workload.turns_hi": "1", "workload.slo_offset_ms": "400", "workload.seed": "41",
    "grid.model_preset": "7b",
}
REPREFILL_7B = merged(MIXED_DRIFT, sim__instances=1, sim__disagg="temporal", sim__controller="false",
                      sim__initial_short_instances=-1, workload__lambda_per_ms=0.01, sim__duration_ms=60000)
LMSYS_32B = {  # config 4: mixed LMsys-like, 32B, graphs on
    "sim.policy": "laps", "sim.disagg": "temporal", "sim.instances": "1", "sim.duration_ms": "60000",
    "sim.slo_ms": "400", "workload.lambda_per_ms": "0.02", "workload.short_fraction": "0.63",
    "workload.short_fraction_later": "0.81", "workload.short_lo": "8", "workload.short_hi": "255",
    "workload.long_lo": "1025", "workload.long_hi": "4096", "workload.turns_lo": "1", "workload.turns_hi": "6",
    "workload.slo_offset_ms": "400", "workload.seed": "7", "grid.model_preset": "32b",
}
SPATIAL_32B = merged(MIXED_DRIFT, grid__model_preset="32b", workload__lambda_per_ms=0.32)

BASELINE_CONFIGS = {
    "c1_default_tiny": DEFAULT,
    "c2_short_7b": SHORT_7B,
    "c3_reprefill_7b": REPREFILL_7B,
    "c4_lmsys_32b": LMSYS_32B,
    "c5_spatial_32b": SPATIAL_32B,
}

# Engine parity matrix: every policy / mode / feature the reference engine has.
PARITY = {
    "default": DEFAULT,
    "mixed_drift": MIXED_DRIFT,
    "c9_spatial_ctrl": {
        "sim.policy": "laps", "sim.disagg": "spatial", "sim.instances": "4", "sim.controller": "true",
        "sim.duration_ms": "12000", "workload.lambda_per_ms": "0.2", "workload.short_fraction": "0.9",
        "workload.short_fraction_later": "0.9", "workload.short_lo": "16", "workload.short_hi": "255",
        "workload.long_lo": "1800", "workload.long_hi": "2200", "workload.seed": "77"},
    "c9_temporal_chunking": {
        "sim.policy": "laps", "sim.disagg": "temporal", "sim.instances": "1", "sim.duration_ms": "20000",
        "workload.lambda_per_ms": "0.02", "workload.short_fraction": "0.63",
        "workload.short_fraction_later": "0.63", "workload.short_lo": "16", "workload.short_hi": "255",
        "workload.long_lo": "1800", "workload.long_hi": "2200", "workload.slo_offset_ms": "400",
        "workload.seed": "78"},
    "fcfs_unified": merged(DEFAULT, sim__policy="fcfs_unified", sim__controller="false",
                           sim__initial_short_instances=-1, sim__instances=2, sim__duration_ms=20000),
    "bucket_no_disagg": merged(DEFAULT, sim__policy="bucket_no_disagg", sim__controller="false",
                               sim__initial_short_instances=-1, sim__instances=3, sim__duration_ms=20000),
    "deadline_free_temporal": merged(DEFAULT, sim__disagg="temporal", sim__instances=1, sim__controller="false",
                                     sim__initial_short_instances=-1, sched__mode="deadline_free",
                                     workload__lambda_per_ms=0.1, sim__duration_ms=20000),
    "spatial_startup_delay": merged(DEFAULT, sim__controller="false", sim__startup_delay_ms=250,
                                    sim__instances=3, workload__lambda_per_ms=0.06, sim__duration_ms=20000),
    "overload_spatial8": merged(MIXED_DRIFT, workload__lambda_per_ms=0.3, sim__duration_ms=20000),
    "graphs_disabled": merged(DEFAULT, grid__mem_budget_mb=100, sim__duration_ms=20000),
    "drift_two_streams": merged(DEFAULT, workload2__lambda_per_ms=0.05, workload2__short_fraction=0.95,
                                workload2__shift_ms=10000, workload2__seed=5, sim__duration_ms=20000),
    **{k: v for k, v in BASELINE_CONFIGS.items() if k != "c1_default_tiny"},
}
