"""Python host-side mirror of the C ABI (include/laps_prefill.h).

`PrefillInstance.forward(shape, members, token_ids)` is the B200 replacement
for the reference's forward stand-in
`batch_service_time(shape, members, cost, overheads)`
(/root/reference/proj/src/cost_model.cpp:128-148): same inputs — a
`BatchShape{l_pad, depth, kind}` and one `(L, H)` row per member — widened
with request/session identity and token ids, returning the measured service
time in ms (plus first tokens / logits on request). Errors mirror the
reference: `ShapeMismatch` for a member longer than `l_pad` or more members
than `depth` (cost_model.cpp:131-139), `ConfigError` for bad descriptors.
"""
from __future__ import annotations

import ctypes
import sys as _sys
from dataclasses import dataclass

import numpy as np

from . import _native as N

KIND_GRAPH, KIND_STANDARD, KIND_PACKED = 0, 1, 2


class ShapeMismatch(N.NativeError):
    pass


class ConfigError(N.NativeError):
    pass


def _check(code: int) -> None:
    if code == -1:
        raise ShapeMismatch(code, N.lib().lp_last_error().decode())
    if code == -2:
        raise ConfigError(code, N.lib().lp_last_error().decode())
    N.check(code)


@dataclass(frozen=True)
class ModelConfig:
    hidden: int
    intermediate: int
    layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    rope_theta: float = 1e6
    rms_eps: float = 1e-6
    init_std: float = 0.02
    weight_seed: int = 1234

    def desc(self) -> N.ModelDesc:
        return N.ModelDesc(self.hidden, self.intermediate, self.layers, self.n_q_heads, self.n_kv_heads,
                           self.head_dim, self.vocab, self.rope_theta, self.rms_eps, self.init_std,
                           self.weight_seed)

    def with_layers(self, layers: int) -> "ModelConfig":
        from dataclasses import replace
        return replace(self, layers=layers)

    # per-forward algorithmic work
    @property
    def weight_bytes(self) -> int:
        h, i, d = self.hidden, self.intermediate, self.head_dim
        per_layer = (self.n_q_heads + 2 * self.n_kv_heads) * d * h + self.n_q_heads * d * h + 3 * h * i
        return 2 * per_layer * self.layers

    @property
    def params_nonembed(self) -> int:
        return self.weight_bytes // 2

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * 2 * self.layers


TINY = ModelConfig(hidden=256, intermediate=704, layers=2, n_q_heads=4, n_kv_heads=2, head_dim=64, vocab=1024)
QWEN25_7B = ModelConfig(hidden=3584, intermediate=18944, layers=28, n_q_heads=28, n_kv_heads=4, head_dim=128,
                        vocab=152064)
QWEN25_32B = ModelConfig(hidden=5120, intermediate=27648, layers=64, n_q_heads=40, n_kv_heads=8, head_dim=128,
                         vocab=152064)
MODELS = {"tiny": TINY, "qwen2.5-7b": QWEN25_7B, "qwen2.5-32b": QWEN25_32B}


@dataclass
class Member:
    """One batch row: prefillsim MemberShape (L, H) plus identity."""
    req_id: int
    session_id: int
    new_tokens: int
    history: int


def synth_token(seed: int, session: int, pos: int, vocab: int) -> int:
    return N.lib().lp_synth_token(seed, session, pos, vocab)


class PrefillInstance:
    """One B200 prefill instance (one reference `Inst`, sim.cpp:95-112)."""

    def __init__(self, model: ModelConfig, device: int = 0, max_tokens: int = 16384, max_members: int = 64,
                 kv_pages: int = 0, use_graphs: bool = True):
        self.model = model
        self._h = ctypes.c_void_p()
        d = N.InstanceDesc(device, 64, kv_pages, max_tokens, max_members, 1 if use_graphs else 0)
        md = model.desc()
        _check(N.lib().lp_instance_create(ctypes.byref(md), ctypes.byref(d), ctypes.byref(self._h)))
        self._last_n = 0

    def close(self) -> None:
        if self._h:
            _check(N.lib().lp_instance_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        # Never touch the CUDA runtime while the interpreter is finalising (its
        # own teardown may already be in progress); the process exit frees it.
        if _sys.is_finalizing():
            return
        try:
            self.close()
        except Exception:
            pass

    def capture_graphs(self, lengths=(8, 16, 32, 64, 128, 256), depths=(1, 2, 4, 8, 16, 32, 64)) -> None:
        L = (ctypes.c_int64 * len(lengths))(*lengths)
        D = (ctypes.c_int32 * len(depths))(*depths)
        _check(N.lib().lp_capture_graphs(self._h, L, len(lengths), D, len(depths)))

    def submit(self, l_pad: int, depth: int, kind: int, members: list[Member], token_ids: np.ndarray) -> None:
        shape = N.Shape(l_pad, depth, kind)
        arr = (N.Member * len(members))(*[N.Member(m.req_id, m.session_id, m.new_tokens, m.history, 1, 0)
                                          for m in members])
        toks = np.ascontiguousarray(token_ids, dtype=np.int32)
        _check(N.lib().lp_submit(self._h, ctypes.byref(shape), arr, len(members),
                                 toks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        self._last_n = len(members)

    def submit_async(self, l_pad: int, depth: int, kind: int, members: list[Member], token_ids: np.ndarray) -> int:
        """Queue a forward without waiting; returns its ticket (lp_submit_async)."""
        shape = N.Shape(l_pad, depth, kind)
        arr = (N.Member * len(members))(*[N.Member(m.req_id, m.session_id, m.new_tokens, m.history, 1, 0)
                                          for m in members])
        toks = np.ascontiguousarray(token_ids, dtype=np.int32)
        t = ctypes.c_int64()
        _check(N.lib().lp_submit_async(self._h, ctypes.byref(shape), arr, len(members),
                                       toks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(t)))
        self._last_n = len(members)
        return t.value

    def ticket_done(self, ticket: int) -> bool:
        d = ctypes.c_int32()
        _check(N.lib().lp_ticket_query(self._h, ticket, ctypes.byref(d)))
        return bool(d.value)

    def ticket_wait(self, ticket: int) -> float:
        ms = ctypes.c_double()
        _check(N.lib().lp_ticket_wait(self._h, ticket, ctypes.byref(ms)))
        return ms.value

    def ticket_tokens(self, ticket: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int32)
        _check(N.lib().lp_ticket_tokens(self._h, ticket, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n))
        return out

    def wait(self) -> float:
        ms = ctypes.c_double()
        _check(N.lib().lp_wait(self._h, ctypes.byref(ms)))
        return ms.value

    def forward(self, l_pad: int, depth: int, kind: int, members: list[Member], token_ids: np.ndarray) -> float:
        self.submit(l_pad, depth, kind, members, token_ids)
        return self.wait()

    def next_tokens(self) -> np.ndarray:
        out = np.empty(self._last_n, dtype=np.int32)
        _check(N.lib().lp_read_next_tokens(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                           self._last_n))
        return out

    def logits(self) -> np.ndarray:
        out = np.empty((self._last_n, self.model.vocab), dtype=np.float32)
        _check(N.lib().lp_read_logits(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.size))
        return out

    def session_pages(self, session_id: int) -> tuple[list[int], int]:
        cap = 4096
        pages = (ctypes.c_int32 * cap)()
        n = ctypes.c_int32()
        kv = ctypes.c_int64()
        _check(N.lib().lp_session_pages(self._h, session_id, pages, cap, ctypes.byref(n), ctypes.byref(kv)))
        return list(pages[: n.value]), kv.value

    def release(self, session_id: int) -> None:
        _check(N.lib().lp_session_release(self._h, session_id))

    def read_kv(self, session_id: int, layer: int, pos0: int, n: int) -> tuple[np.ndarray, np.ndarray]:
        m = self.model
        k = np.empty((n, m.n_kv_heads, m.head_dim), dtype=np.uint16)
        v = np.empty_like(k)
        _check(N.lib().lp_read_kv(self._h, session_id, layer, pos0, n, k.ctypes.data, v.ctypes.data))
        return k, v

    def last_io(self) -> tuple[int, int]:
        """(H2D bytes of the last submit, D2H bytes of the last first-token read)."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(N.lib().lp_last_io(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def last_launches(self) -> int:
        """Kernels the last submit put on the GPU (graph nodes or eager launches)."""
        n = ctypes.c_int32()
        _check(N.lib().lp_last_launches(self._h, ctypes.byref(n)))
        return n.value

    def timer_record(self, slot: int) -> None:
        _check(N.lib().lp_timer_record(self._h, slot))

    def timer_elapsed(self, a: int, b: int) -> float:
        ms = ctypes.c_double()
        _check(N.lib().lp_timer_elapsed(self._h, a, b, ctypes.byref(ms)))
        return ms.value

    def time_gemm(self, layer: int, which: int, t_cap: int, n_live: int, iters: int = 20) -> float:
        """Average ms of one projection GEMM (0 qkv, 1 o, 2 gate/up, 3 down)
        with this instance's weights and launch plan (CUDA events)."""
        ms = ctypes.c_double()
        _check(N.lib().lpk_time_gemm(self._h, layer, which, t_cap, n_live, iters, ctypes.byref(ms)))
        return ms.value

    def attention_schedule(self) -> tuple[int, int, int]:
        """(pieces, split units merged in-kernel, CTAs with work) of the last
        submit's tcgen05 attention (test hook, laps_prefill_testing.h)."""
        a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(N.lib().lpk_last_attention_schedule(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    @staticmethod
    def migrate(src: "PrefillInstance", dst: "PrefillInstance", session_id: int) -> None:
        _check(N.lib().lp_session_migrate(src._h, dst._h, session_id))
