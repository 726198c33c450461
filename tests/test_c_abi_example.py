"""The drop-in boundary from plain C: examples/laps_simulate.c links
liblaps_prefill.so and drives the engine (include/laps_engine.h) and a GPU
prefill instance (include/laps_prefill.h) the way the reference's own
`prefillsim simulate` CLI runs (tools/main.cpp:76-93). Cost-model mode must
reproduce the reference's events.log / metrics.json for configs/default.cfg
byte for byte; replay mode on a B200 must keep the
same bytes while executing every dispatch."""
import hashlib
import json
import subprocess
from pathlib import Path

import pytest

from paper_2601_11589_b200 import build as B
from paper_2601_11589_b200 import scenarios as S

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "build" / "examples" / "laps_simulate"
DEFAULT_EVENTS = "0455c026730291d46246e0670a7c5e77d866853c01e3778a1012c52c2afac081"
DEFAULT_METRICS = "f0f3e3cafaf4d447140346f8c3ce6263a05afb72ad9585011489b76f8d2420d1"


def _run(tmp_path, mode, model="tiny"):
    if not EXE.exists():
        B.build_examples()
    cfg = tmp_path / "default.cfg"
    cfg.write_text(S.text(S.DEFAULT))
    out = tmp_path / mode
    r = subprocess.run([str(EXE), str(cfg), str(out), mode, model], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1]), out


def _sha(p):
    return hashlib.sha256(p.read_bytes()).hexdigest()


def test_c_program_cost_model_matches_reference(tmp_path):
    st, out = _run(tmp_path, "cost")
    assert st["dispatches"] == 3517 and st["gpu_forwards"] == 0
    assert _sha(out / "events.log") == DEFAULT_EVENTS
    assert _sha(out / "metrics.json") == DEFAULT_METRICS


def test_c_program_rejects_bad_config(tmp_path):
    if not EXE.exists():
        B.build_examples()
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("sim.instances = 0\n")
    r = subprocess.run([str(EXE), str(cfg), str(tmp_path / "o"), "cost"], capture_output=True, text=True)
    assert r.returncode == 1 and "instance" in r.stderr


@pytest.mark.gpu
def test_c_program_replay_on_gpu(tmp_path):
    st, out = _run(tmp_path, "replay")
    assert st["gpu_forwards"] == 3517
    assert _sha(out / "events.log") == DEFAULT_EVENTS
