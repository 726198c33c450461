"""Single-request goldens pinned by the reference's own unit tests
(/root/reference/proj/tests/test_sim.cpp:193-241, :497-507), replayed through
this framework's host engine (C ABI lp_sim_run, cost-model mode) with the
tests' example cost parameters (test_sim.cpp:20-27)."""
import json

import pytest

from paper_2601_11589_b200 import engine as E

EXAMPLE_COST = "cost.alpha = 1e-5\ncost.beta = 0.01\ncost.gamma_w = 0.02\ncost.gamma_r = 0.002\n"


def run(tmp_path, reqs, extra=""):
    tr = tmp_path / "trace.jsonl"
    tr.write_text("".join(json.dumps(r) + "\n" for r in reqs))
    out = tmp_path / "out"
    st = E.simulate(f"trace.path = {tr}\n" + EXAMPLE_COST + extra, "", out)
    log = [json.loads(l) for l in (out / "events.log").read_text().splitlines()]
    metrics = json.loads((out / "metrics.json").read_text())
    return st, log, metrics


LONE = {"session_id": 0, "turn": 1, "arrival_ms": 0, "new_tokens": 100}


def test_lone_packed_request_takes_its_service_time(tmp_path):
    # test_sim.cpp:193-207: 0.5 launch + 1.1 compute + 2.0 cache write
    st, log, m = run(tmp_path, [LONE], "sim.policy = fcfs_unified\n")
    assert len(log) == 3 and log[1]["reason"] == "fcfs_pack" and log[1]["t"] == 0
    assert log[2]["t"] == pytest.approx(3.6, rel=1e-12)
    assert st.ttft_mean_ms == pytest.approx(3.6, rel=1e-12)
    assert m["overall"]["mean_wait_ms"] == 0


def test_idle_adaptive_stream_dispatches_at_window_expiry(tmp_path):
    # test_sim.cpp:209-228
    st, log, m = run(tmp_path, [LONE])
    d = log[1]
    assert (d["t"], d["reason"], d["graph"], d["l_pad"], d["depth"], d["real"], d["padded"]) == \
        (50.0, "window_expired", 1, 128, 1, 100, 128)
    assert log[2]["service"] == pytest.approx(4.05384, rel=1e-12)
    assert st.ttft_mean_ms == pytest.approx(54.05384, rel=1e-12)
    assert m["overall"]["padding_overhead"] == pytest.approx(0.28)
    assert m["overall"]["graph_hit_rate"] == 1.0


def test_imminent_deadline_pulls_dispatch_forward(tmp_path):
    # test_sim.cpp:230-241: window (20-1)-5 = 14, slack 5 <= sigma -> sla_break
    st, log, _ = run(tmp_path, [{**LONE, "deadline_ms": 20.0}])
    assert log[1]["t"] == pytest.approx(14) and log[1]["reason"] == "sla_break"
    assert st.ttft_mean_ms == pytest.approx(18.05384, rel=1e-12)


def test_startup_delay_defers_first_dispatch(tmp_path):
    # test_sim.cpp:497-507
    st, log, _ = run(tmp_path, [LONE], "sim.policy = fcfs_unified\nsim.startup_delay_ms = 10\n")
    assert log[1]["t"] == pytest.approx(10)
    assert st.ttft_mean_ms == pytest.approx(13.6, rel=1e-12)


def test_empty_stream_controller_ticks_once(tmp_path):
    # test_sim.cpp:243-257
    st, log, _ = run(tmp_path, [], "sim.disagg = spatial\nsim.instances = 2\nsim.controller = true\n")
    assert len(log) == 1 and log[0]["kind"] == "controller_tick"
    assert st.arrivals == 0 and st.completed == 0


def test_long_chunk_chain(tmp_path):
    # chunking semantics (scheduler.cpp:322-338): 700 tokens -> 512 + 188, back to back
    st, log, _ = run(tmp_path, [{**LONE, "new_tokens": 700}])
    ds = [r for r in log if r["kind"] == "dispatch"]
    assert [(d["chunk"], d["chunks"], d["real"]) for d in ds] == [(1, 2, 512), (2, 2, 188)]
    comp = [r for r in log if r["kind"] == "batch_complete"]
    assert ds[1]["t"] == comp[0]["t"] and [c["final"] for c in comp] == [0, 1]
