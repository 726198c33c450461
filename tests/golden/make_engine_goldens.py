"""Regenerate tests/golden/engine_digests.json from the REFERENCE build.

Runs the unmodified reference engine (oracle/_ref/libprefillsim_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile) on every scenario
in paper_2601_11589_b200.scenarios.PARITY and records the sha256 of its
events.log / metrics.json plus line counts. Only runnable where
/root/reference exists (this container); the digests travel with the repo.
"""
import ctypes
import hashlib
import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import scenarios as S  # noqa: E402

REF = ROOT / "oracle" / "_ref" / "libprefillsim_ref.so"


def ref_lib():
    if not REF.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    L = ctypes.CDLL(str(REF))
    L.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.ref_last_error.restype = ctypes.c_char_p
    return L


def run_ref(cfg: dict, out: Path):
    L = ref_lib()
    secs, nd = ctypes.c_double(), ctypes.c_int64()
    rc = L.ref_simulate(S.text(cfg).encode(), b"", str(out).encode(), ctypes.byref(secs), ctypes.byref(nd))
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return secs.value, nd.value


def digest(p: Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


if __name__ == "__main__":
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, cfg in S.PARITY.items():
            d = Path(td) / name
            secs, nd = run_ref(cfg, d)
            out[name] = {"events_sha256": digest(d / "events.log"), "metrics_sha256": digest(d / "metrics.json"),
                         "events_lines": len((d / "events.log").read_text().splitlines()), "dispatches": nd}
            print(name, out[name], f"{secs*1e3:.1f} ms", flush=True)
    (ROOT / "tests" / "golden" / "engine_digests.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
