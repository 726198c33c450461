"""tcgen05 GEMM parity vs a torch fp32 reference of the same op (bf16 inputs,
fp32 accumulate). Tolerance: relative Frobenius error < 2e-3 and max-abs
within bf16 output rounding."""
import ctypes

import pytest
import torch

from paper_2601_11589_b200 import _native as N

pytestmark = pytest.mark.gpu


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def run_gemm(M, Ntok, K, splits=1, mode=0, bn=None, bias=False, n_live=None, seed=0, pair=1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = (torch.randn(M, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(Ntok, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(M, device="cuda", generator=g) * 0.1).bfloat16() if bias else None
    bn = bn or next(b for b in (16, 32, 64, 128, 256) if b >= min(Ntok, 256))
    ref = X.float() @ W.float().t()  # [N, M]
    if b is not None:
        ref = ref + b.float()
    nd = None
    if n_live is not None:
        nd = torch.tensor([n_live], dtype=torch.int32, device="cuda")
    ws = None
    if mode == 1:
        ws = torch.zeros(splits, Ntok, M, device="cuda", dtype=torch.float32)
        out = None
        ldo = M
    elif mode == 2:
        out = torch.zeros(Ntok, M // 2, device="cuda", dtype=torch.bfloat16)
        ldo = M // 2
    elif mode == 3:
        out = torch.zeros(Ntok, M, device="cuda", dtype=torch.float32)
        ldo = M
    else:
        out = torch.zeros(Ntok, M, device="cuda", dtype=torch.bfloat16)
        ldo = M
    rc = N.lib().lpk_gemm(_ptr(W), _ptr(X), _ptr(out) if out is not None else None,
                          _ptr(ws) if ws is not None else None, _ptr(b) if b is not None else None,
                          M, Ntok, K, splits, mode, bn, ldo, _ptr(nd) if nd is not None else None, None, pair)
    N.check(rc)
    torch.cuda.synchronize()
    if mode == 1:
        got = ws.sum(0)
    elif mode == 2:
        g_ = ref[:, 0::2].bfloat16().float()
        u_ = ref[:, 1::2].bfloat16().float()
        ref = torch.nn.functional.silu(g_) * u_
        got = out.float()
    else:
        got = out.float()
    return got, ref


def _close(got, ref, n_live=None):
    if n_live is not None:
        got, ref = got[:n_live], ref[:n_live]
    rel = (got - ref).norm() / ref.norm().clamp_min(1e-6)
    assert rel < 5e-3, f"rel err {rel}"


@pytest.mark.parametrize("M,Ntok,K", [(128, 16, 64), (256, 8, 512), (384, 100, 1024), (1024, 256, 3584),
                                      (512, 600, 512), (4608, 64, 3584)])
def test_gemm_bf16(M, Ntok, K):
    got, ref = run_gemm(M, Ntok, K, bias=True)
    _close(got, ref)


@pytest.mark.parametrize("splits", [2, 5])
def test_gemm_splitk(splits):
    got, ref = run_gemm(3584, 200, 3584, splits=splits, mode=1)
    _close(got, ref)


def test_gemm_silu_mul():
    got, ref = run_gemm(1536, 40, 256, mode=2)
    _close(got, ref)


def test_gemm_f32_and_live_count():
    got, ref = run_gemm(1024, 256, 512, mode=3, n_live=77)
    _close(got, ref, n_live=77)
    assert torch.all(got[80:] == 0)


@pytest.mark.parametrize("M,Ntok,K,bn,mode,splits", [(256, 128, 512, 128, 0, 1), (512, 256, 1024, 256, 0, 1),
                                                      (3584, 300, 3584, 256, 1, 3), (1536, 200, 256, 256, 2, 1),
                                                      (4608, 64, 3584, 64, 1, 4), (1024, 1000, 512, 128, 3, 1)])
def test_gemm_pair(M, Ntok, K, bn, mode, splits):
    """cta_group::2 variant (CTA pair, M = 256 per pair, B split over the pair)."""
    got, ref = run_gemm(M, Ntok, K, splits=splits, mode=mode, bn=bn, pair=2, bias=(mode == 0))
    _close(got, ref)


def test_gemm_pair_live_count():
    got, ref = run_gemm(1024, 512, 512, mode=3, bn=256, pair=2, n_live=300)
    _close(got, ref, n_live=300)


@pytest.mark.parametrize("M,Ntok,K,bn,mode,splits,pair,n_live", [
    (1024, 256, 512, 256, 3, 1, 2, 187),    # one tile, MMA N = 192
    (1024, 512, 512, 256, 3, 1, 2, 385),    # two balanced tiles of 208
    (1536, 1024, 256, 256, 2, 1, 2, 777),   # SiLU epilogue, 4 tiles of 208
    (3584, 256, 3584, 256, 1, 3, 2, 130),   # split-K partials, N = 144
    (1024, 64, 512, 64, 1, 2, 2, 17),       # pair, N = 32 (16 rows per CTA)
    (1024, 128, 512, 128, 0, 1, 1, 33),     # single CTA, N = 48
    (1024, 2048, 512, 256, 3, 1, 2, 2047),  # 8 tiles of 256, last one N = 256 with 255 live
])
def test_gemm_dynamic_tile_width(M, Ntok, K, bn, mode, splits, pair, n_live):
    """Token tiles sized from the live count (balanced widths, MMA N rounded to 16)."""
    got, ref = run_gemm(M, Ntok, K, splits=splits, mode=mode, bn=bn, pair=pair, n_live=n_live, bias=(mode == 0))
    _close(got, ref, n_live=n_live)
    if mode in (0, 3):
        assert torch.all(got[n_live:] == 0)


@pytest.mark.parametrize("M,Ntok,K,bn,pair,n_live,max_ctas", [
    (7168, 512, 5120, 256, 2, None, 0),    # 32B QKV at a 512-token chunk: 56 tiles on 74 pairs
    (5120, 512, 5120, 256, 2, 500, 0),     # 32B O, live count below capacity
    (5120, 512, 27648, 256, 2, None, 0),   # 32B down projection
    (256, 64, 4096, 64, 1, None, 148),     # 2 tiles of 64 K blocks on 148 CTAs: 64 segments per tile
    (1024, 600, 3584, 128, 2, 517, 20),    # 10 pairs, ragged live count
])
def test_gemm_stream_k(M, Ntok, K, bn, pair, n_live, max_ctas):
    """Stream-K (csrc/gemm_sm100.cu): equal (weight tile, K-block) shares per
    group of CTAs (pairs), one member per token tile; segment j of a tile lands in ws slice j and the segment counts in
    the table the reduction kernels read. Summing each element's segments in
    slice order reproduces the GEMM, every tile is covered, and the output is
    bitwise reproducible run to run."""
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(M, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(Ntok, K, device="cuda", generator=g).bfloat16()
    live = n_live or Ntok
    ref = X.float()[:live] @ W.float().t()
    nd = torch.tensor([live], dtype=torch.int32, device="cuda")
    workers = (max_ctas or torch.cuda.get_device_properties(0).multi_processor_count) // pair
    nt = -(-live // bn)
    tw = min(bn, (-(-live // nt) + 15) // 16 * 16)
    tiles_n = -(-live // tw)
    m_tiles = M // (128 * pair)
    groups = workers // tiles_n  # one CTA (pair) per token tile, in lockstep
    total = m_tiles * (K // 64)
    per = -(-total // groups)
    slices = (K // 64 - 1) // per + 2
    ws = torch.full((slices, Ntok, M), float("nan"), device="cuda", dtype=torch.float32)
    tab = torch.full((4 + (M // 128) * (-(-Ntok // 16)),), -1, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(3):
        N.check(N.lib().lpk_gemm_stream_k(_ptr(W), _ptr(X), _ptr(ws), M, Ntok, K, bn, pair, _ptr(nd),
                                          _ptr(tab), max_ctas, None))
        torch.cuda.synchronize()
        assert tab[:3].tolist() == [tw, tiles_n, 128 * pair]
        nseg = tab[4:4 + m_tiles * tiles_n].view(m_tiles, tiles_n)
        assert int(nseg.min()) >= 1 and int(nseg.max()) <= slices
        # one extra segment per share boundary that falls inside a weight tile
        assert int(nseg.sum()) - m_tiles * tiles_n == tiles_n * sum(1 for j in range(1, groups)
                                                                    if j * per < total and (j * per) % (K // 64))
        # element (t, f) sums the slices of its tile's segments, in order
        per_elem = nseg.repeat_interleave(128 * pair, 0).repeat_interleave(tw, 1)[:M, :live].t()
        out = ws[0, :live].clone()
        for s_ in range(1, slices):
            out = torch.where(per_elem > s_, out + ws[s_, :live], out)
        outs.append(out)
    _close(outs[0], ref)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
