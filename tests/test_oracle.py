"""The CPU oracle itself (CPU only): the page-allocator restatement, and
properties of the forward restatement checked against independent
evaluations (fp64 softmax attention, causality, chunking invariance)."""
import math

import numpy as np
import pytest
import torch

from oracle import forward_oracle as FO
from oracle.pages import PAGE, PageOracle


def test_page_oracle_lowest_first_and_release():
    p = PageOracle(8)
    p.submit([(1, 100, 0), (2, 10, 0)])          # 2 pages + 1 page
    assert p.table(1) == ([0, 1], 100) and p.table(2) == ([2], 10)
    p.submit([(1, 30, 100)])                     # 130 tokens -> 3 pages
    assert p.table(1) == ([0, 1, 3], 130)
    p.release(1)
    p.submit([(3, 64 * 3, 0)])                   # reuses 0, 1, 3 in that order
    assert p.table(3) == ([0, 1, 3], 192)
    with pytest.raises(ValueError):
        p.submit([(4, 5, 10)])                   # history not resident
    with pytest.raises(MemoryError):
        p.submit([(5, PAGE * 6, 0)])


@pytest.fixture(scope="module")
def tiny():
    return FO.OracleModel(FO.TINY)


def test_tiled_attention_matches_fp64_softmax(tiny):
    """The oracle's 64-key-tile online softmax (bf16 P) is within bf16
    rounding of an exact fp64 causal GQA attention."""
    s = tiny.s
    g = torch.Generator().manual_seed(0)
    H, L = 150, 40
    q = torch.randn(L, s.n_q_heads, s.head_dim, generator=g)
    K = torch.randn(H + L, s.n_kv_heads, s.head_dim, generator=g)
    V = torch.randn(H + L, s.n_kv_heads, s.head_dim, generator=g)
    got = tiny.attend(q, K, V, H)
    G = s.n_q_heads // s.n_kv_heads
    Kh, Vh = K.double().repeat_interleave(G, 1), V.double().repeat_interleave(G, 1)
    sc = torch.einsum("qhd,khd->hqk", q.double(), Kh) / math.sqrt(s.head_dim)
    mask = torch.arange(H + L)[None, :] > torch.arange(H, H + L)[:, None]
    sc = sc.masked_fill(mask[None], float("-inf"))
    want = torch.einsum("hqk,khd->qhd", torch.softmax(sc, -1), Vh).reshape(L, -1)
    assert (got.double() - want).abs().max().item() < 2e-2


def test_chunked_prefill_equals_single_prefill():
    """Chunk k of a long prefill sees history H + (k-1)*C_l
    (scheduler.cpp:322-338): two chunks reproduce one prefill."""
    a, b = FO.OracleModel(FO.TINY), FO.OracleModel(FO.TINY)
    toks = FO.tokens(7, 9, 0, 300, FO.TINY.vocab)
    one = a.forward([(9, 300, 0)], [toks])
    b.forward([(9, 200, 0)], [toks[:200]])
    two = b.forward([(9, 100, 200)], [toks[200:]])
    assert (one - two).abs().max().item() < 2e-2
    Ka, _ = a.read_kv(9, 1, 0, 300)
    Kb, _ = b.read_kv(9, 1, 0, 300)
    assert (Ka - Kb).abs().max().item() < 2e-2


def test_batch_composition_invariance(tiny):
    """A member's logits do not depend on its batch mates."""
    o1, o2 = FO.OracleModel(FO.TINY), FO.OracleModel(FO.TINY)
    t1 = FO.tokens(7, 1, 0, 50, FO.TINY.vocab)
    t2 = FO.tokens(7, 2, 0, 80, FO.TINY.vocab)
    alone = o1.forward([(1, 50, 0)], [t1])
    batched = o2.forward([(2, 80, 0), (1, 50, 0)], [t2, t1])
    assert (alone[0] - batched[1]).abs().max().item() < 1e-4


def test_history_must_be_resident(tiny):
    with pytest.raises(ValueError):
        FO.OracleModel(FO.TINY).forward([(3, 10, 5)], [np.zeros(10, np.int32)])


def test_rope_is_a_rotation(tiny):
    x = torch.randn(5, tiny.s.n_q_heads, tiny.s.head_dim)
    pos = torch.tensor([0, 1, 17, 1000, 65535])
    y = tiny.rope(x, pos)
    assert torch.allclose(y.norm(dim=-1), x.norm(dim=-1), rtol=1e-5)
    assert torch.allclose(y[0], x[0])  # position 0 is the identity


def test_streaming_oracle_matches_resident_weights():
    """stream=True (one layer's weights at a time, layer-major over a sequence
    of forwards) is the same computation as the resident-weight oracle."""
    import torch
    a, b = FO.OracleModel(FO.TINY), FO.OracleModel(FO.TINY, stream=True)
    t1, t2, t3 = (FO.tokens(7, 0, 0, 50, 1024), FO.tokens(7, 0, 50, 20, 1024), FO.tokens(7, 1, 0, 33, 1024))
    r1 = a.forward([(0, 50, 0), (1, 33, 0)], [t1, t3])
    r2 = a.forward([(0, 20, 50)], [t2])
    s1, s2 = b.forward_seq([([(0, 50, 0), (1, 33, 0)], [t1, t3]), ([(0, 20, 50)], [t2])])
    assert torch.equal(r1, s1) and torch.equal(r2, s2)
    for l in range(FO.TINY.layers):
        assert torch.equal(a.read_kv(0, l, 0, 70)[0], b.read_kv(0, l, 0, 70)[0])
