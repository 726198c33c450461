"""CPU tests of the GEMM launch planner (executor.cu plan_gemm / choose_tiles
through lpk_plan_gemm): the tile and split-K choices the chunk and bucket
forwards run, the split bound, and that the planner charges each extra
split its fp32 partial round trip (profiles/r02_tile_sweep.txt,
profiles/r02_decompose_chunk_after_planner.txt)."""
import ctypes

import pytest

from paper_2601_11589_b200 import _native as N

SHAPES = {  # (M out, K in) of the projections
    "qkv32": (7168, 5120), "o32": (5120, 5120), "gu32": (55296, 5120), "down32": (5120, 27648),
    "qkv7": (4608, 3584), "o7": (3584, 3584), "gu7": (37888, 3584), "down7": (3584, 18944),
}


def plan(M, K, t_cap, n_live, sms=148, allow_split=True):
    f = N.lib().lpk_plan_gemm
    f.restype = ctypes.c_int32
    f.argtypes = [ctypes.c_int32] * 6 + [ctypes.POINTER(ctypes.c_int32)] * 4
    out = [ctypes.c_int32() for _ in range(4)]
    N.check(f(M, K, t_cap, n_live, sms, 1 if allow_split else 0, *[ctypes.byref(o) for o in out]))
    return tuple(o.value for o in out)  # bn, pair, n_tiles, splits


def test_chunk_plans_512_tokens():
    # 512-token chunks: QKV and O run one K slice (5 slices made the reduction
    # read 73 MB of partials); the deep-K down projection runs stream-K
    # (splits -1: equal K shares per CTA pair; 5 slices before, -10 %).
    assert plan(*SHAPES["qkv32"], 512, 512) == (256, 2, 2, 1)
    assert plan(*SHAPES["o32"], 512, 512)[2:] == (3, 1)
    assert plan(*SHAPES["down32"], 512, 512)[2:] == (2, -1)
    assert plan(*SHAPES["down7"], 384, 384)[3] == -1
    assert plan(*SHAPES["qkv7"], 512, 512)[3] == 1


def test_stream_k_window():
    # offered only between one and three 256-token tiles, never for fused
    # epilogues (allow_split = 0) nor for weight-streaming batches
    for name, (M, K) in SHAPES.items():
        for t in (16, 128, 255, 256, 1024, 4096):
            assert plan(M, K, t, t)[3] != -1
        assert plan(M, K, 512, 512, allow_split=False)[3] == 1


def test_split_bounds_and_fused_epilogues():
    for name, (M, K) in SHAPES.items():
        for t in (16, 64, 256, 512, 1024, 4096):
            for n in sorted({1, t // 2, t}):
                bn, pair, nt, s = plan(M, K, t, n)
                assert s == -1 or (1 <= s <= 8 and s <= max(1, (K // 64) // 4) and s * t <= max(8192, t))
                assert pair in (1, 2) and bn in (16, 32, 64, 128, 256) and nt >= 1
                assert plan(M, K, t, n, allow_split=False)[3] == 1


def test_weight_streaming_batches_fill_the_sms():
    # A 16-token graph bucket of the 32B QKV (56 row tiles, no CTA pair) splits
    # K so the units cover the 148 SMs.
    bn, pair, nt, s = plan(*SHAPES["qkv32"], 16, 12)
    assert (bn, pair, nt) == (16, 1, 1) and 56 * s >= 148 * 0.75


@pytest.mark.parametrize("t", [256, 384, 512])
def test_partial_traffic_is_charged(t):
    # More live tokens make every extra split dearer (its partial grows with
    # n_live), so the chosen split count never grows with n_live at a fixed
    # capacity.
    M, K = SHAPES["qkv32"]
    assert 1 <= plan(M, K, t, t)[3] <= plan(M, K, t, t // 2 + 128)[3]
