"""Second compute-sanitizer workload (round 2): the ticketed asynchronous
boundary (several lp_submit_async in flight, results read through tickets),
asynchronous session migration / copy followed by forwards on both
instances, the engine's REPLAY and WALL modes over two instances, and the
tcgen05 attention (head_dim 128) with key splits merged in-kernel — on a
small model whose GEMMs stay below 128-token tiles (no CTA pairs), so
racecheck can run the whole workload.
usage: compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize_run2.py"""
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200 import engine as E  # noqa: E402
from paper_2601_11589_b200 import scenarios as S  # noqa: E402
from paper_2601_11589_b200.instance import (KIND_GRAPH, KIND_STANDARD, TINY, Member, ModelConfig,  # noqa: E402
                                            PrefillInstance)

rng = np.random.default_rng(0)
m = ModelConfig(hidden=512, intermediate=1024, layers=2, n_q_heads=4, n_kv_heads=1, head_dim=128, vocab=1024)
a = PrefillInstance(m, max_tokens=1024, max_members=8, kv_pages=128)
b = PrefillInstance(m, max_tokens=1024, max_members=8, kv_pages=128)
a.capture_graphs(lengths=(16, 64), depths=(1, 2))
tok = lambda n: rng.integers(0, m.vocab, n).astype(np.int32)  # noqa: E731
# history of 1536 tokens in 64-token eager chunks (tcgen05 attention, growing key ranges)
tickets = []
for p in range(0, 1536, 64):
    tickets.append(a.submit_async(64, 1, KIND_STANDARD, [Member(p, 7, 64, p)], tok(64)))
for t in tickets[-12:]:
    a.ticket_wait(t)
print("history ok", a.ticket_tokens(tickets[-1], 1), flush=True)
# short re-prefill over the long history through a graph (key splits, merge)
t1 = a.submit_async(16, 2, KIND_GRAPH, [Member(0, 7, 12, 1536), Member(1, 8, 16, 0)], tok(28))
PrefillInstance.migrate(a, b, 8)                      # async: ordered after t1
t2 = b.submit_async(16, 1, KIND_GRAPH, [Member(2, 8, 9, 16)], tok(9))
print("migrate ok", a.ticket_tokens(t1, 2), b.ticket_tokens(t2, 1), flush=True)
a.close()
b.close()
# the tier engine on two tiny instances: REPLAY (async, concurrent) and WALL clock
insts = [PrefillInstance(TINY, max_tokens=2048, max_members=64, kv_pages=2000) for _ in range(2)]
for i in insts:
    i.capture_graphs(lengths=(16, 64, 256), depths=(1, 2, 4))
cfg = S.merged(S.DEFAULT, sim__instances=2, sim__controller="false", sim__initial_short_instances=1,
               sim__duration_ms=800, workload__lambda_per_ms=0.05, workload__seed=3)
d = Path(tempfile.mkdtemp())
st = E.simulate(S.text(cfg), "", d / "replay", mode=E.REPLAY, instances=insts, token_seed=7)
sw = E.simulate(S.text(cfg), "", d / "wall", mode=E.WALL, instances=insts, token_seed=7)
print("engine ok", st.gpu_forwards, st.kv_migrations, sw.completed, sw.kv_migrations, flush=True)
for i in insts:
    i.close()
