"""Multi-instance (N > 1) host logic on CPU with world_size-2 gloo.

Each rank is an independent prefill instance behind the length-aware router
(spatial disaggregation: no collective on the data path). Every rank runs the
host engine on its own request stream (seed 41 + rank, as bench.py does), and
the job-level numbers use bench.py's own aggregation: requests summed over
ranks, time = max over ranks. The test checks that against each rank's
single-process result."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    cfg = bench.scenario(rank, lam=0.3, dur=3000)
    st = E.simulate(S.text(cfg))  # cost-model clock: deterministic per rank
    value, total, t_max = bench.aggregate_throughput(dist, st.completed, st.active_ms, rank)
    q.put((rank, st.completed, st.active_ms, value, total, t_max))
    dist.destroy_process_group()


def test_two_rank_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, c0, a0, v0, tot0, tm0), (r1, c1, a1, v1, tot1, tm1) = res
    assert c0 > 0 and c1 > 0 and c0 != c1           # independent streams
    assert tot0 == tot1 == c0 + c1
    assert tm0 == tm1 == max(a0, a1)
    assert v0 == pytest.approx((c0 + c1) / (max(a0, a1) / 1000.0))
