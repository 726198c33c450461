"""CPU-side checks of the C-ABI library (no GPU calls): it loads, exports every
symbol include/*.h declares, and its host-callable generators agree bit for
bit with the oracle's C restatement."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import forward_oracle as FO
from paper_2601_11589_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]


def _declared(header: Path) -> list[str]:
    text = header.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|const char\*|uint16_t)\s+(lpk?_\w+)\s*\(", text, re.M)))


@pytest.mark.parametrize("header", ["laps_prefill.h", "laps_engine.h", "laps_prefill_testing.h"])
def test_every_declared_symbol_is_exported(header):
    lib = N.lib()
    names = _declared(ROOT / "include" / header)
    assert names, header
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"{header}: not exported: {missing}"


def test_symbol_lists_match_headers():
    assert set(N.PUBLIC_SYMBOLS) == set(_declared(ROOT / "include" / "laps_prefill.h"))
    assert set(N.ENGINE_SYMBOLS) == set(_declared(ROOT / "include" / "laps_engine.h"))


def test_version_and_error_channel():
    assert b"sm_100a" in N.lib().lp_version()
    assert isinstance(N.lib().lp_last_error(), bytes)


def test_token_generator_matches_oracle():
    L = N.lib()
    rng = np.random.default_rng(0)
    for seed, vocab in ((7, 1024), (7, 152064), (12345, 151936)):
        sess = rng.integers(0, 1 << 40, 16)
        pos = rng.integers(0, 1 << 20, 16)
        for s, p in zip(sess, pos):
            want = FO.tokens(seed, int(s), int(p), 1, vocab)[0]
            assert L.lp_synth_token(seed, int(s), int(p), vocab) == want


def test_weight_generator_matches_oracle_bit_for_bit():
    L = N.lib()
    L.lpk_synth_weight_bits.restype = ctypes.c_uint16
    L.lpk_synth_weight_bits.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float]
    scale = float(np.float32(np.float32(0.02) * np.float32(np.sqrt(3.0))) / np.float32(8388608.0))
    import torch
    for tid in (1, 2, 1000, 1003, 1004, 1016 + 5):
        flat = FO.weight_bf16(3, 67, 1234, tid, scale).view(torch.int16).numpy().view(np.uint16).reshape(-1)
        for idx in (0, 1, 66, 67, 150, 200):
            assert L.lpk_synth_weight_bits(1234, tid, idx, scale) == flat[idx]


def test_interleaved_gate_up_layout_matches_oracle():
    """The device stores gate/up row-interleaved (row 2j = gate j, 2j+1 = up j);
    the oracle's interleave option must produce the same bits."""
    import torch
    scale = 1e-7
    inter = FO.weight_bf16(8, 16, 99, 1003, scale, interleave=True).view(torch.int16).numpy()
    gate = FO.weight_bf16(4, 16, 99, 1003, scale).view(torch.int16).numpy()
    up = FO.weight_bf16(4, 16, 99, 1004, scale).view(torch.int16).numpy()
    assert (inter[0::2] == gate).all() and (inter[1::2] == up).all()
