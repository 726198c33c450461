"""ctypes loader for the in-tree native library (liblaps_prefill.so).

The product path is native only: if the library is missing, importing the
bindings raises — there is no Python or CPU fallback for any kernel.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "liblaps_prefill.so"

_lib = None


class NativeError(RuntimeError):
    """A negative LP_ERR_* status from the C ABI."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


ERR_NAMES = {-1: "LP_ERR_SHAPE", -2: "LP_ERR_CONFIG", -3: "LP_ERR_OOM", -4: "LP_ERR_CUDA",
             -5: "LP_ERR_STATE", -9: "LP_ERR_INTERNAL"}


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA extension is required; there is no fallback)")
        _lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
        _declare(_lib)
    return _lib


def check(code: int) -> int:
    if code < 0:
        msg = lib().lp_last_error().decode(errors="replace")
        raise NativeError(code, f"{ERR_NAMES.get(code, code)}: {msg}")
    return code


c_i32, c_i64, c_u64, c_f32, c_f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double
vp = ctypes.c_void_p


class ModelDesc(ctypes.Structure):
    _fields_ = [("hidden", c_i32), ("intermediate", c_i32), ("layers", c_i32),
                ("n_q_heads", c_i32), ("n_kv_heads", c_i32), ("head_dim", c_i32), ("vocab", c_i32),
                ("rope_theta", c_f32), ("rms_eps", c_f32), ("init_std", c_f32),
                ("weight_seed", c_u64)]


class InstanceDesc(ctypes.Structure):
    _fields_ = [("device", c_i32), ("page_size", c_i32), ("kv_pages", c_i64),
                ("max_tokens", c_i64), ("max_members", c_i32), ("use_graphs", c_i32)]


class Shape(ctypes.Structure):
    _fields_ = [("l_pad", c_i64), ("depth", c_i32), ("kind", c_i32)]


class Member(ctypes.Structure):
    _fields_ = [("req_id", c_i64), ("session_id", c_i64), ("new_tokens", c_i64),
                ("history", c_i64), ("want_logits", c_i32), ("reserved", c_i32)]


# Every symbol include/laps_prefill.h declares (checked by the CPU tests).
PUBLIC_SYMBOLS = [
    "lp_instance_create", "lp_instance_destroy", "lp_capture_graphs", "lp_submit", "lp_wait",
    "lp_read_next_tokens", "lp_read_logits", "lp_session_pages", "lp_session_release",
    "lp_read_kv", "lp_session_migrate", "lp_synth_token", "lp_last_error", "lp_version",
    "lp_instance_model", "lp_timer_record", "lp_timer_elapsed", "lp_last_io", "lp_last_launches",
    "lp_submit_async", "lp_ticket_query", "lp_ticket_wait", "lp_ticket_tokens", "lp_session_copy",
]
ENGINE_SYMBOLS = ["lp_sim_run", "lp_sim_run_ex", "lp_sim_trace", "lp_sim_sweep"]  # include/laps_engine.h


def _declare(L: ctypes.CDLL) -> None:
    def sig(name, res, *args):
        if hasattr(L, name):
            f = getattr(L, name)
            f.restype = res
            f.argtypes = list(args)

    sig("lp_last_error", ctypes.c_char_p)
    sig("lp_version", ctypes.c_char_p)
    sig("lp_synth_token", c_i32, c_u64, c_i64, c_i64, c_i32)
    sig("lp_instance_create", c_i32, ctypes.POINTER(ModelDesc), ctypes.POINTER(InstanceDesc),
        ctypes.POINTER(vp))
    sig("lp_instance_destroy", c_i32, vp)
    sig("lp_capture_graphs", c_i32, vp, ctypes.POINTER(c_i64), c_i32, ctypes.POINTER(c_i32), c_i32)
    sig("lp_submit", c_i32, vp, ctypes.POINTER(Shape), ctypes.POINTER(Member), c_i32,
        ctypes.POINTER(c_i32))
    sig("lp_wait", c_i32, vp, ctypes.POINTER(c_f64))
    sig("lp_submit_async", c_i32, vp, ctypes.POINTER(Shape), ctypes.POINTER(Member), c_i32,
        ctypes.POINTER(c_i32), ctypes.POINTER(c_i64))
    sig("lp_ticket_query", c_i32, vp, c_i64, ctypes.POINTER(c_i32))
    sig("lp_ticket_wait", c_i32, vp, c_i64, ctypes.POINTER(c_f64))
    sig("lp_ticket_tokens", c_i32, vp, c_i64, ctypes.POINTER(c_i32), c_i32)
    sig("lp_read_next_tokens", c_i32, vp, ctypes.POINTER(c_i32), c_i32)
    sig("lp_read_logits", c_i32, vp, ctypes.POINTER(c_f32), ctypes.c_size_t)
    sig("lp_session_pages", c_i32, vp, c_i64, ctypes.POINTER(c_i32), c_i32, ctypes.POINTER(c_i32),
        ctypes.POINTER(c_i64))
    sig("lp_session_release", c_i32, vp, c_i64)
    sig("lp_read_kv", c_i32, vp, c_i64, c_i32, c_i64, c_i64, vp, vp)
    sig("lp_session_migrate", c_i32, vp, vp, c_i64)
    sig("lp_session_copy", c_i32, vp, vp, c_i64)
    sig("lp_instance_model", c_i32, vp, ctypes.POINTER(ModelDesc))
    sig("lp_timer_record", c_i32, vp, c_i32)
    sig("lp_last_io", c_i32, vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64))
    sig("lp_last_launches", c_i32, vp, ctypes.POINTER(c_i32))
    sig("lp_timer_elapsed", c_i32, vp, c_i32, c_i32, ctypes.POINTER(c_f64))
    sig("lpk_time_gemm", c_i32, vp, c_i32, c_i32, c_i32, c_i32, c_i32, ctypes.POINTER(c_f64))
    sig("lpk_last_attention_schedule", c_i32, vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), ctypes.POINTER(c_i32))
    # kernel-level test hooks (include/laps_prefill_testing.h)
    sig("lpk_gemm", c_i32, vp, vp, vp, vp, vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, vp, vp, c_i32)
    sig("lpk_gemm_stream_k", c_i32, vp, vp, vp, c_i32, c_i32, c_i32, c_i32, c_i32, vp, vp, c_i32, vp)
