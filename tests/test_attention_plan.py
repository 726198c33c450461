"""CPU tests of the persistent tcgen05 attention's host planner
(csrc/host/attn_plan.cpp through lpk_plan_attention): coverage, list
balance, merge bookkeeping and the whole-unit fallback, on the chunk shapes
the c4 bench runs (Qwen2.5-32B: GQA group 5, 8 KV heads; Qwen2.5-7B: group
7, 4 KV heads) and on random block sets."""
import ctypes

import numpy as np
import pytest

from paper_2601_11589_b200 import _native as N

PIECE_COST = 1.5  # kAttnPieceCost


def plan(needs, nkv, ncta=148):
    L = N.lib()
    f = L.lpk_plan_attention
    f.restype = ctypes.c_int32
    f.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                  ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                  ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    arr = (ctypes.c_int32 * len(needs))(*needs)
    cap = 8 * len(needs) * nkv + 4 * ncta
    out = (ctypes.c_int32 * (6 * cap))()
    n, m = ctypes.c_int32(), ctypes.c_int32()
    lc, span = ctypes.c_double(), ctypes.c_double()
    N.check(f(arr, len(needs), nkv, ncta, out, cap, ctypes.byref(n), ctypes.byref(m), ctypes.byref(lc),
              ctypes.byref(span)))
    pieces = np.frombuffer(out, dtype=np.int32)[: 6 * n.value].reshape(-1, 6)
    return pieces, m.value, lc.value, span.value


def chunk_needs(H, L=512, G=5):
    rows = L * G
    needs = [(H + min(r0 + 127, rows - 1) // G + 1 + 63) // 64 for r0 in range(0, rows, 128)]
    return sorted(needs, reverse=True)


def check(needs, nkv, ncta=148):
    pieces, merges, cap, span = plan(needs, nkv, ncta)
    # every (block, head) unit is covered exactly once, by contiguous page ranges
    for b, need in enumerate(needs):
        for g in range(nkv):
            sel = pieces[(pieces[:, 1] == b) & (pieces[:, 2] == g)]
            rng = sorted((int(p[3]), int(p[4])) for p in sel)
            assert rng[0][0] == 0 and rng[-1][1] == need
            assert all(rng[k][1] == rng[k + 1][0] for k in range(len(rng) - 1))
            # a split unit shares one merge entry, a whole unit has none
            cis = {int(p[5]) for p in sel}
            assert (len(sel) > 1) == (cis != {-1}) and len(cis) == 1
    assert merges == len({int(p[5]) for p in pieces if p[5] >= 0})
    assert pieces[:, 0].min() >= 0 and pieces[:, 0].max() < ncta
    load = np.zeros(ncta)
    for p in pieces:
        load[p[0]] += (p[4] - p[3] + 1) // 2 + PIECE_COST
    return pieces, merges, cap, span, load


@pytest.mark.parametrize("H", [0, 512, 2048, 4096, 8192, 16384])
def test_32b_chunk_lists(H):
    needs = chunk_needs(H)
    pieces, merges, cap, span, load = check(needs, nkv=8)
    unit = max((n + 1) // 2 for n in needs) + PIECE_COST
    if span < 0:  # split lists chosen: balanced to the McNaughton capacity
        assert load.max() <= cap + 1.0
        assert load.max() < 0.75 * 2 * unit  # 160 units on 148 SMs took 2 unit-lengths before
        assert merges > 0
    else:         # whole units: longest-first makespan, no merges
        assert merges == 0 and load.max() == pytest.approx(span)
    if H >= 2048:
        assert span < 0  # long histories are worth splitting (profiles/r02_attn_experiments.md)


@pytest.mark.parametrize("H", [0, 2048, 3584])
def test_7b_chunk_keeps_whole_units(H):
    """112 units for 148 SMs: splitting does not pay at these histories, so
    every unit runs whole on its own list (the round-1 grid's schedule)."""
    needs = chunk_needs(H, G=7)
    pieces, merges, cap, span, load = check(needs, nkv=4)
    assert span >= 0 and merges == 0
    assert len(pieces) == len(needs) * 4 and len(set(pieces[:, 0])) == len(pieces)


def test_random_block_sets():
    rng = np.random.default_rng(0)
    for _ in range(40):
        nb = int(rng.integers(1, 60))
        needs = sorted((int(x) for x in rng.integers(1, 300, nb)), reverse=True)
        nkv = int(rng.choice([1, 2, 4, 8]))
        ncta = int(rng.choice([8, 37, 148]))
        pieces, merges, cap, span, load = check(needs, nkv, ncta)
        if span < 0:
            assert load.max() <= cap + 1.0
