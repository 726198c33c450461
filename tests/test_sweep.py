"""`prefillsim sweep` (tools/main.cpp:114-168) on the framework's engine:
sweep.csv must be byte-identical to the reference library driven the same way
(oracle/ref_driver.cpp ref_sweep, the CLI restated on the unmodified library),
and a sweep that executes every dispatch on the GPU (replay mode) must produce
the same bytes."""
import ctypes
from pathlib import Path

import pytest

from paper_2601_11589_b200 import engine as E
from paper_2601_11589_b200 import scenarios as S

ROOT = Path(__file__).resolve().parents[1]
REF_LIB = ROOT / "oracle" / "_ref" / "libprefillsim_ref.so"
BASE = S.merged(S.DEFAULT, sim__duration_ms=8000)

CASES = [("short_concurrency", [2.0, 0.5, 1.0]), ("sched.w_max_ms", [10, 50]), ("sim.instances", [2, 4])]


@pytest.mark.skipif(not REF_LIB.exists(), reason="reference oracle not built (needs /root/reference)")
@pytest.mark.parametrize("param,values", CASES)
def test_sweep_csv_matches_reference(tmp_path, param, values):
    ours = E.sweep(S.text(BASE), param, values, tmp_path / "ours")
    L = ctypes.CDLL(str(REF_LIB))
    L.ref_sweep.argtypes = [ctypes.c_char_p] * 5
    vals = ",".join(repr(float(v)) for v in values)
    assert L.ref_sweep(S.text(BASE).encode(), b"", str(tmp_path / "ref").encode(), param.encode(), vals.encode()) == 0
    ref = (tmp_path / "ref" / "sweep.csv").read_bytes()
    assert ours.read_bytes() == ref
    assert ref.count(b"\n") == len(values) + 1


def test_sweep_rejects_empty_values(tmp_path):
    from paper_2601_11589_b200 import _native as N
    with pytest.raises(N.NativeError):
        E.sweep(S.text(BASE), "short_concurrency", [], tmp_path)


@pytest.mark.gpu
def test_sweep_replay_on_gpu_keeps_bytes(tmp_path):
    from paper_2601_11589_b200.instance import TINY, PrefillInstance
    inst = PrefillInstance(TINY, max_tokens=4096, max_members=64, kv_pages=2048)
    inst.capture_graphs()
    cost = E.sweep(S.text(BASE), "short_concurrency", [0.5, 1.0], tmp_path / "cost")
    gpu = E.sweep(S.text(BASE), "short_concurrency", [0.5, 1.0], tmp_path / "gpu", mode=E.REPLAY, instances=[inst])
    assert gpu.read_bytes() == cost.read_bytes()
    inst.close()
