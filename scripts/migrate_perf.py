"""Session-KV migration throughput (lp_session_migrate, the spatial-mode
exchange of SURVEY.md §8(e)): two Qwen2.5-7B-shaped instances; a session
with H resident tokens moves from one to the other. On one GPU the page-gather
kernel copies inside HBM; across GPUs the same kernel reads the peer's pool
over NVLink. Prints ms and GB/s (H x 56 KiB)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_11589_b200.instance import KIND_STANDARD, QWEN25_7B, Member, PrefillInstance  # noqa: E402

m = QWEN25_7B
a = PrefillInstance(m, max_tokens=4096, max_members=8, kv_pages=4096)
b = PrefillInstance(m, max_tokens=4096, max_members=8, kv_pages=4096)
rng = np.random.default_rng(0)
for H in (512, 2048, 8192, 32768):
    ts, dev = [], []
    for it in range(4):
        sid = 1000 * H + it
        for p in range(0, H, 4096):
            n = min(4096, H - p)
            a.forward(n, 1, KIND_STANDARD, [Member(0, sid, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))
        torch.cuda.synchronize()
        b.timer_record(0)
        t0 = time.perf_counter()
        PrefillInstance.migrate(a, b, sid)
        ts.append(time.perf_counter() - t0)
        b.timer_record(1)
        dev.append(b.timer_elapsed(0, 1))
        b.release(sid)
    t = float(np.median(ts[1:]))
    byts = H * m.kv_bytes_per_token
    td = float(np.median(dev[1:])) / 1e3
    print(f"H={H:5d}: {byts / 1e6:8.1f} MB  host {t * 1e3:7.3f} ms ({byts / t / 1e9:6.1f} GB/s)  "
          f"device {td * 1e3:7.3f} ms ({byts / td / 1e9:6.1f} GB/s moved, {2 * byts / td / 1e9:6.1f} GB/s HBM r+w)")
