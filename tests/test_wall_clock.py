"""Wall-clock engine (LP_SIM_WALL) on CPU: forwards emulated by sleeping for
their cost-model service time (no GPU), two spatial instances.

Checks what the virtual clock cannot: the two instances serve concurrently
(their busy time adds up to more than the elapsed time), arrivals are
released in real time, and the TTFT reported is measured on steady_clock.
"""
import json

import pytest

from paper_2601_11589_b200 import engine as E
from paper_2601_11589_b200 import scenarios as S

SPATIAL2 = S.merged(S.DEFAULT, sim__instances=2, sim__controller="false", sim__initial_short_instances=1,
                    sim__duration_ms=1500, workload__lambda_per_ms=0.2, workload__seed=11,
                    workload__long_lo=300, workload__long_hi=600)


def _records(path):
    return [json.loads(x) for x in path.read_text().splitlines()]


def test_wall_clock_instances_overlap(tmp_path):
    cm = E.simulate(S.text(SPATIAL2), "", tmp_path / "cm", mode=E.COST_MODEL)
    st = E.simulate(S.text(SPATIAL2), "", tmp_path / "wall", mode=E.WALL)
    assert st.arrivals == cm.arrivals
    assert st.completed == cm.completed == st.arrivals  # every request is served
    recs = _records(tmp_path / "wall" / "events.log")
    busy = {0: 0.0, 1: 0.0}
    for r in recs:
        if r["kind"] == "batch_complete":
            busy[r["inst"]] += r["service"]
    assert busy[0] > 0 and busy[1] > 0
    # Both lanes were busy at the same time: total service exceeds the span.
    span = max(r["t"] for r in recs) - min(r["t"] for r in recs)
    assert busy[0] + busy[1] > 1.3 * span, (busy, span)
    # The run took real time: at least the stream's duration.
    assert st.engine_wall_s * 1000 >= 0.9 * max(r["t"] for r in recs if r["kind"] == "arrival")


def test_wall_clock_ttft_tracks_cost_model(tmp_path):
    cfg = S.merged(SPATIAL2, workload__lambda_per_ms=0.02)  # light load: TTFT ~ service time
    cm = E.simulate(S.text(cfg), "", tmp_path / "cm", mode=E.COST_MODEL)
    st = E.simulate(S.text(cfg), "", tmp_path / "wall", mode=E.WALL)
    assert st.completed == cm.completed
    # Same service times, same policy; wall time adds only host lag (sleep
    # granularity), so the medians agree to within a few ms.
    assert st.ttft_p50_ms == pytest.approx(cm.ttft_p50_ms, abs=5.0)
    assert st.ttft_p50_ms >= cm.ttft_p50_ms - 0.5
    recs = _records(tmp_path / "wall" / "events.log")
    arrivals = [r for r in recs if r["kind"] == "arrival"]
    dispatch_t = {}
    for r in recs:
        if r["kind"] == "dispatch":
            for q in r["reqs"]:
                dispatch_t.setdefault(q, r["t"])
    # Nothing is dispatched before it arrived (real-time release).
    for a in arrivals:
        if a["req"] in dispatch_t:
            assert dispatch_t[a["req"]] >= a["t"] - 1e-6


def test_wall_clock_needs_handles_for_gpu_modes(tmp_path):
    with pytest.raises(Exception):
        E.simulate(S.text(SPATIAL2), "", tmp_path, mode=E.REPLAY)  # REPLAY needs instances
