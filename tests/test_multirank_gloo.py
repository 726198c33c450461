"""Multi-GPU (N > 1) host logic on CPU with world_size-2 gloo.

bench.py under torchrun: rank 0 drives every GPU from one host engine (the
reference's length-aware router is global, sim.cpp:379-411) and the other
ranks only join the barriers. Here rank 0 runs bench.scenario(2, ...) — the
2-GPU spatial configuration — on the wall-clock engine with paced (sleeping)
forwards, rank 1 idles, and the test checks the spatial split: short work on
the short-pool instance, long chunks on the long-pool one, both busy at the
same time, plus the window accounting bench.py reports."""
import json
import os
import socket
import tempfile
from pathlib import Path

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank))
    import bench
    dist = bench.dist_init(ws)
    bench.barrier(dist)
    if rank == 0:
        from paper_2601_11589_b200 import engine as E
        from paper_2601_11589_b200 import scenarios as S
        cfg = bench.scenario(2, 0.01, 1200)
        out = Path(tempfile.mkdtemp())
        st = E.simulate(S.text(cfg), "", out, mode=E.WALL)
        recs = [json.loads(x) for x in (out / "events.log").read_text().splitlines()]
        q.put((rank, st.arrivals, st.completed, recs, cfg))
    else:
        q.put((rank, 0, 0, [], {}))
    bench.barrier(dist)
    dist.destroy_process_group()


def test_two_rank_spatial_router():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, arrivals, completed, recs, cfg = res[0]
    assert cfg["sim.disagg"] == "spatial" and cfg["sim.instances"] == "2"
    assert arrivals > 0 and completed == arrivals
    disp = [r for r in recs if r["kind"] == "dispatch"]
    assert {r["inst"] for r in disp if r["reason"] != "long_chunk"} == {0}   # short pool
    assert {r["inst"] for r in disp if r["reason"] == "long_chunk"} == {1}   # long pool
    assert res[1][1] == 0  # rank 1 did no work


def test_window_accounting():
    import bench
    disp = [{"reason": "long_chunk", "chunk": 1, "chunks": 4, "reqs": [3]},
            {"reason": "depth_reached", "reqs": [5, 6]},
            {"reason": "long_chunk", "chunk": 4, "chunks": 4, "reqs": [3]}]
    assert bench.request_equivalents(disp) == pytest.approx(2.5)
