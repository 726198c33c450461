"""TEST INFRASTRUCTURE — CPU oracle for the prefill forward.

Parity status: **parity unpinned** for logits / KV values. The reference
(prefillsim) has no model, tokens, weights or KV cache (SURVEY.md §0.1,
/root/reference/SPEC.md:14); its "forward" is the closed form
`batch_service_time` (/root/reference/proj/src/cost_model.cpp:128-148). This
module is the builder-defined restatement that the CUDA path is checked
against, and it follows the reference only where the reference speaks:

  * which tokens a forward covers: new L tokens attend causally to H cached
    tokens plus themselves — the alpha*L*(L+2H) term (cost_model.cpp:36-41,
    PAPER.md:141-152);
  * chunk k of a long prefill sees history H + (k-1)*C_l
    (scheduler.cpp:322-338);
  * dummy pad rows (sim.cpp:249-253) and the pad tail produce nothing.

Everything else is the Qwen2 decoder definition (RMSNorm, QKV with bias,
rotate-half RoPE theta=1e6, GQA, SiLU-gated MLP, untied LM head) evaluated in
fp32 with bf16 rounding at the same storage points as the kernels:
normed activations, q/k/v, the attention output, the gate/up projections and
the SiLU*up product are rounded to bf16; the residual stream stays fp32.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
SYNTH_LIB = HERE / "_build" / "libsynth_ref.so"

# Tensor ids — restated from paper_2601_11589_b200/csrc/executor.cu.
TID_EMBED, TID_LM_HEAD = 1, 2
TID_LAYER_BASE, TID_LAYER_STRIDE = 1000, 16
T_QKV, T_QKV_BIAS, T_O, T_GATE, T_UP, T_DOWN = 0, 1, 2, 3, 4, 5

_synth = None


def synth_lib() -> ctypes.CDLL:
    global _synth
    if _synth is None:
        if not SYNTH_LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "synth"], check=True)
        _synth = ctypes.CDLL(str(SYNTH_LIB))
        _synth.oracle_token.restype = ctypes.c_int32
        _synth.oracle_token.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
        _synth.oracle_tokens.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int32, ctypes.c_void_p]
        _synth.oracle_weights_bf16.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_float, ctypes.c_int]
        _synth.oracle_weights_bf16_mt.argtypes = _synth.oracle_weights_bf16.argtypes + [ctypes.c_int]
    return _synth


def tokens(seed: int, session: int, pos0: int, n: int, vocab: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    synth_lib().oracle_tokens(seed, session, pos0, n, vocab, out.ctypes.data)
    return out


def weight_bf16(rows: int, cols: int, seed: int, tid: int, scale: float, interleave: bool = False,
                row0: int = 0, nrows: int | None = None) -> torch.Tensor:
    """bf16 weight tensor (as torch.bfloat16) from the counter-based generator."""
    nrows = rows if nrows is None else nrows
    buf = np.empty((nrows, cols), dtype=np.uint16)
    synth_lib().oracle_weights_bf16_mt(buf.ctypes.data, row0, nrows, cols, seed, tid, ctypes.c_float(scale),
                                       1 if interleave else 0, os.cpu_count() or 1)
    return torch.from_numpy(buf.view(np.int16)).view(torch.bfloat16)


def bf16r(x: torch.Tensor) -> torch.Tensor:
    """Round fp32 to bf16 (RNE) and back."""
    return x.to(torch.bfloat16).to(torch.float32)


@dataclass
class ModelSpec:
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

    @property
    def qkv_out(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim


class OracleModel:
    """fp32 CPU restatement of the Qwen2-style prefill forward.

    stream=True never holds more than one decoder layer's weights: each
    forward_seq() call regenerates layer l from the counter RNG, runs layer l
    of every batch it was given (in order — batch k+1's layer l only needs
    batch k's layer-l KV), and drops it. That makes full-depth Qwen2.5-32B
    checks fit in host memory (one fp32 layer = 2 GB instead of 125 GB)."""

    def __init__(self, spec: ModelSpec, threads: int | None = None, stream: bool = False):
        if threads:
            torch.set_num_threads(threads)
        self.s = spec
        s = spec
        scale = float(np.float32(np.float32(s.init_std) * np.float32(math.sqrt(3.0))) / np.float32(8388608.0))
        self.scale = scale
        self.stream = stream
        self.layers = None if stream else [self.layer_weights(l) for l in range(s.layers)]
        emb_scale = float(np.float32(math.sqrt(3.0)) / np.float32(8388608.0))
        self.embed = weight_bf16(s.vocab, s.hidden, s.weight_seed, TID_EMBED, emb_scale).float()
        self.lm_head = weight_bf16(s.vocab, s.hidden, s.weight_seed, TID_LM_HEAD, scale).float()
        d = s.head_dim
        self.inv_freq = torch.tensor(
            [np.float32(1.0 / math.pow(float(np.float32(s.rope_theta)), (2.0 * i) / d)) for i in range(d // 2)],
            dtype=torch.float32)
        # Logical KV per session: list over layers of (K, V) [pos, nkv, d] fp32 (bf16 values).
        self.kv: dict[int, list[list[torch.Tensor]]] = {}

    def layer_weights(self, l: int) -> dict:
        s, scale, seed = self.s, self.scale, self.s.weight_seed
        base = TID_LAYER_BASE + TID_LAYER_STRIDE * l
        return {
            "wqkv": weight_bf16(s.qkv_out, s.hidden, seed, base + T_QKV, scale).float(),
            "bqkv": weight_bf16(1, s.qkv_out, seed, base + T_QKV_BIAS, scale).float()[0],
            "wo": weight_bf16(s.hidden, s.n_q_heads * s.head_dim, seed, base + T_O, scale).float(),
            "wgate": weight_bf16(s.intermediate, s.hidden, seed, base + T_GATE, scale).float(),
            "wup": weight_bf16(s.intermediate, s.hidden, seed, base + T_UP, scale).float(),
            "wd": weight_bf16(s.hidden, s.intermediate, seed, base + T_DOWN, scale).float(),
        }

    # -- building blocks ----------------------------------------------------
    def rmsnorm(self, x: torch.Tensor) -> torch.Tensor:
        var = (x * x).mean(-1, keepdim=True)
        return bf16r(x * torch.rsqrt(var + self.s.rms_eps))  # gamma == 1

    def rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        half = self.s.head_dim // 2
        ang = pos.to(torch.float32)[:, None] * self.inv_freq[None, :]  # [T, d/2]
        cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        x0, x1 = x[..., :half], x[..., half:]
        return torch.cat([x0 * cos - x1 * sin, x1 * cos + x0 * sin], dim=-1)

    ATTN_TILE = 64  # keys per online-softmax step (one KV page)

    def attend(self, q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, H: int) -> torch.Tensor:
        """Causal GQA attention of L new queries (positions H..H+L-1) over
        K/V [H+L, nkv, d]. Softmax is evaluated online over 64-key tiles in
        the log2 domain with the probabilities rounded to bf16 before the
        P.V product — the bf16 storage point every flash-style kernel has."""
        s = self.s
        nq, nkv, d = s.n_q_heads, s.n_kv_heads, s.head_dim
        G = nq // nkv
        L = q.shape[0]
        scale_log2 = float(np.float32(1.4426950408889634 / math.sqrt(d)))
        Kh = K.repeat_interleave(G, dim=1)  # [S, nq, d]
        Vh = V.repeat_interleave(G, dim=1)
        qpos = torch.arange(H, H + L)[:, None]
        m = torch.full((nq, L), float("-inf"))
        lsum = torch.zeros(nq, L)
        o = torch.zeros(nq, L, d)
        for k0 in range(0, H + L, self.ATTN_TILE):
            k1 = min(k0 + self.ATTN_TILE, H + L)
            sc = torch.einsum("qhd,khd->hqk", q, Kh[k0:k1])
            kpos = torch.arange(k0, k1)[None, :]
            sc = sc.masked_fill((kpos > qpos)[None], float("-inf"))
            m_new = torch.maximum(m, sc.amax(-1) * scale_log2)
            corr = torch.exp2(m - m_new)
            p = torch.exp2(sc * scale_log2 - m_new[..., None])
            lsum = lsum * corr + p.sum(-1)
            o = o * corr[..., None] + torch.einsum("hqk,khd->hqd", bf16r(p), Vh[k0:k1])
            m = m_new
        return (o / lsum[..., None]).permute(1, 0, 2).reshape(L, nq * d)

    def kv_len(self, session: int) -> int:
        c = self.kv.get(session)
        return 0 if c is None else c[0][0].shape[0]

    # -- the forward --------------------------------------------------------
    def forward(self, members: list[tuple[int, int, int]], toks: list[np.ndarray]) -> torch.Tensor:
        """members: (session, new_tokens L, history H) in plan order; toks[i]
        are member i's L new token ids. Returns fp32 logits [n, vocab] of the
        last new token per member; updates the logical KV cache."""
        return self.forward_seq([(members, toks)])[0]

    def forward_seq(self, batches: list[tuple[list[tuple[int, int, int]], list[np.ndarray]]]) -> list[torch.Tensor]:
        """Several forwards in submission order, evaluated layer-major (each
        layer's weights are materialised once for all of them)."""
        s = self.s
        states = []
        for members, toks in batches:
            ids = torch.from_numpy(np.concatenate(toks).astype(np.int64))
            x = self.embed[ids].clone()
            states.append({
                "members": members, "x": x, "xn": self.rmsnorm(x),
                "pos": torch.cat([torch.arange(H, H + L) for (_, L, H) in members]),
                "starts": np.cumsum([0] + [L for (_, L, _) in members]),
                "checked": False,
            })
        for l in range(s.layers):
            w = self.layer_weights(l) if self.stream else self.layers[l]
            for st in states:
                if not st["checked"]:  # history residency, at the batch's turn in submission order
                    for (sid, L, H) in st["members"]:
                        if self.kv_len(sid) < H:
                            raise ValueError(f"session {sid}: history {H} not resident ({self.kv_len(sid)})")
                    st["checked"] = True
                self._layer(l, w, st)
            del w
        out = []
        for st in states:
            last = torch.tensor([st["starts"][i + 1] - 1 for i in range(len(st["members"]))])
            out.append(st["xn"][last] @ self.lm_head.t())
        return out

    def _layer(self, l: int, w: dict, st: dict) -> None:
        s = self.s
        nq, nkv, d = s.n_q_heads, s.n_kv_heads, s.head_dim
        members, starts, pos, x, xn = st["members"], st["starts"], st["pos"], st["x"], st["xn"]
        qkv = xn @ w["wqkv"].t() + w["bqkv"]
        q = qkv[:, : nq * d].view(-1, nq, d)
        k = qkv[:, nq * d: (nq + nkv) * d].view(-1, nkv, d)
        v = qkv[:, (nq + nkv) * d:].view(-1, nkv, d)
        q, k, v = bf16r(self.rope(q, pos)), bf16r(self.rope(k, pos)), bf16r(v)
        out = torch.empty(q.shape[0], nq * d)
        for i, (sid, L, H) in enumerate(members):
            a, b = starts[i], starts[i + 1]
            cache = self.kv.setdefault(sid, [[torch.zeros(0, nkv, d), torch.zeros(0, nkv, d)]
                                             for _ in range(s.layers)])
            K0, V0 = cache[l]
            K = torch.cat([K0[:H], k[a:b]], 0)
            V = torch.cat([V0[:H], v[a:b]], 0)
            if K0.shape[0] > H + L:  # keep resident positions beyond this member
                K = torch.cat([K, K0[H + L:]], 0)
                V = torch.cat([V, V0[H + L:]], 0)
            cache[l] = [K, V]
            out[a:b] = bf16r(self.attend(q[a:b], K[: H + L], V[: H + L], H))
        x = x + out @ w["wo"].t()
        xn = self.rmsnorm(x)
        g = bf16r(xn @ w["wgate"].t())
        u = bf16r(xn @ w["wup"].t())
        act = bf16r(torch.nn.functional.silu(g) * u)
        x = x + act @ w["wd"].t()
        st["x"], st["xn"] = x, self.rmsnorm(x)

    def read_kv(self, session: int, layer: int, pos0: int, n: int):
        K, V = self.kv[session][layer]
        return K[pos0: pos0 + n], V[pos0: pos0 + n]


# Builder-defined model shapes (Qwen2.5 public configs).
TINY = ModelSpec(hidden=256, intermediate=704, layers=2, n_q_heads=4, n_kv_heads=2, head_dim=64, vocab=1024)
QWEN25_7B = ModelSpec(hidden=3584, intermediate=18944, layers=28, n_q_heads=28, n_kv_heads=4, head_dim=128,
                      vocab=152064)
QWEN25_32B = ModelSpec(hidden=5120, intermediate=27648, layers=64, n_q_heads=40, n_kv_heads=8, head_dim=128,
                       vocab=152064)


def with_layers(spec: ModelSpec, layers: int) -> ModelSpec:
    from dataclasses import replace
    return replace(spec, layers=layers)
