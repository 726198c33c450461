"""Python mirror of the host engine's C ABI (include/laps_engine.h).

`simulate(config_text, overrides, out_dir)` is the reference's
`prefillsim simulate --config <cfg> --out <dir>` (tools/main.cpp:76-93); with
`mode=REPLAY` / `mode=LIVE` and GPU instances, every dispatch also runs its
real forward on B200 (see laps_engine.h for the three modes).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

from . import _native as N
from .instance import PrefillInstance

COST_MODEL, REPLAY, LIVE, WALL = 0, 1, 2, 3


class SimStats(ctypes.Structure):
    _fields_ = [("arrivals", ctypes.c_int64), ("completed", ctypes.c_int64), ("dispatches", ctypes.c_int64),
                ("gpu_forwards", ctypes.c_int64), ("fill_forwards", ctypes.c_int64),
                ("kv_migrations", ctypes.c_int64), ("real_tokens", ctypes.c_int64),
                ("active_ms", ctypes.c_double), ("ttft_mean_ms", ctypes.c_double),
                ("ttft_p50_ms", ctypes.c_double), ("ttft_p90_ms", ctypes.c_double),
                ("ttft_p99_ms", ctypes.c_double), ("rps", ctypes.c_double), ("slo_violation", ctypes.c_double),
                ("gpu_ms_total", ctypes.c_double), ("engine_wall_s", ctypes.c_double),
                ("window_dispatches", ctypes.c_int64), ("window_requests", ctypes.c_int64),
                ("window_fills", ctypes.c_int64), ("window_kernels", ctypes.c_int64),
                ("window_h2d_bytes", ctypes.c_int64), ("window_d2h_bytes", ctypes.c_int64),
                ("window_device_ms", ctypes.c_double), ("window_wall_ms", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class SimOpts(ctypes.Structure):
    """lp_sim_opts: GPU dispatches [window_first, window_first + window_count)
    form a timed window (REPLAY mode); stop_after_window runs later
    dispatches on the clock only."""
    _fields_ = [("window_first", ctypes.c_int64), ("window_count", ctypes.c_int64),
                ("stop_after_window", ctypes.c_int32), ("reserved", ctypes.c_int32)]


def _declare():
    L = N.lib()
    if not getattr(L, "_engine_declared", False):
        L.lp_sim_run.restype = ctypes.c_int32
        L.lp_sim_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int32,
                                 ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_uint64,
                                 ctypes.POINTER(SimStats)]
        L.lp_sim_run_ex.restype = ctypes.c_int32
        L.lp_sim_run_ex.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_uint64,
                                    ctypes.POINTER(SimOpts), ctypes.POINTER(SimStats)]
        L.lp_sim_sweep.restype = ctypes.c_int32
        L.lp_sim_sweep.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int32,
                                   ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_uint64,
                                   ctypes.c_char_p, ctypes.c_char_p]
        L.lp_sim_trace.restype = ctypes.c_int32
        L.lp_sim_trace.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]
        L._engine_declared = True
    return L


def sweep(config_text: str, param: str, values, out_dir: str | Path, overrides: str | dict = "",
          mode: int = COST_MODEL, instances: list[PrefillInstance] | None = None, token_seed: int = 7) -> Path:
    """The reference CLI's `prefillsim sweep` (tools/main.cpp:114-168): one
    engine run per value of `param` (apply_sweep_param semantics, e.g.
    "short_concurrency" scales workload.lambda_per_ms), in cost-model mode or
    on GPU instances; returns the path of sweep.csv."""
    if isinstance(overrides, dict):
        overrides = "".join(f"{k} = {v}\n" for k, v in overrides.items())
    L = _declare()
    insts = instances or []
    arr = (ctypes.c_void_p * max(1, len(insts)))(*[i._h.value for i in insts])
    vals = ",".join(repr(float(v)) for v in values)
    N.check(L.lp_sim_sweep(config_text.encode(), overrides.encode(), str(out_dir).encode(), mode,
                           arr if insts else None, len(insts), token_seed, param.encode(), vals.encode()))
    return Path(out_dir) / "sweep.csv"


def read_config(path: str | Path) -> str:
    return Path(path).read_text()


def simulate(config_text: str, overrides: str | dict = "", out_dir: str | Path = "", mode: int = COST_MODEL,
             instances: list[PrefillInstance] | None = None, token_seed: int = 7,
             window: tuple[int, int] | None = None, stop_after_window: bool = True) -> SimStats:
    """One engine run (lp_sim_run_ex). `window=(first, count)` times GPU
    dispatches [first, first + count) of a REPLAY run (window_* stats)."""
    if isinstance(overrides, dict):
        overrides = "".join(f"{k} = {v}\n" for k, v in overrides.items())
    L = _declare()
    insts = instances or []
    arr = (ctypes.c_void_p * max(1, len(insts)))(*[i._h.value for i in insts])
    st = SimStats()
    opts = SimOpts(window[0], window[1], 1 if stop_after_window else 0, 0) if window else SimOpts()
    N.check(L.lp_sim_run_ex(config_text.encode(), overrides.encode(), str(out_dir).encode(), mode,
                            arr if insts else None, len(insts), token_seed, ctypes.byref(opts), ctypes.byref(st)))
    return st


def dump_trace(config_text: str, overrides: str | dict, path: str | Path) -> None:
    if isinstance(overrides, dict):
        overrides = "".join(f"{k} = {v}\n" for k, v in overrides.items())
    N.check(_declare().lp_sim_trace(config_text.encode(), overrides.encode(), str(path).encode()))


@dataclass
class TraceRow:
    id: int
    session: int
    turn: int
    L: int
    H: int
    arrival: float
    deadline: float | None


def load_trace_dump(path: str | Path) -> list[TraceRow]:
    rows = []
    for line in Path(path).read_text().splitlines():
        a = line.split()
        rows.append(TraceRow(int(a[0]), int(a[1]), int(a[2]), int(a[3]), int(a[4]), float(a[5]),
                             None if a[6] == "none" else float(a[6])))
    return rows
