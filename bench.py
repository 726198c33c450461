#!/usr/bin/env python3
"""Benchmark: LAPS prefill-instance throughput on B200 (BASELINE.json metric
"prefill req/s and p50/p90 TTFT at 1/2/4/8 B200; HBM GB/s & tensor-pipe %
roofline").

Workload (BASELINE.json configs[1]): Qwen2.5-7B-shaped random-init bf16
decoder, short-prefill-only stream (8-255 new tokens, one turn per session,
400 ms SLO, seed 41 + rank) at high concurrency (lambda = 0.5 req/ms offered
per GPU), served by the LAPS dual-queue / adaptive-wait-depth scheduler on one
temporal instance per GPU. A "step" is one dispatched batch forward (one
per-(l_pad, depth) CUDA-graph replay).

Phases (per rank; N ranks = N independent instances, spatial
disaggregation, no collective on the data path -> "scaling": "weak"):
  A  REPLAY engine run at a saturating 1 req/ms/GPU: the host engine (clock =
     the reference cost model, so batch composition is byte-identical to the
     reference scheduler's) executes every dispatch on the GPU; its dispatch
     sequence is the workload of the timed region. A second, LIVE run at a
     sub-saturation 0.25 req/ms (clock = measured forward times) gives the
     reported TTFT p50/p90.
  B  `value`: W warm-up + K timed steps replaying that dispatch sequence
     through lp_submit back to back; inputs (token ids / page tables) are
     staged by the instance, the timed region is bracketed by CUDA events on
     the instance stream (max over ranks). Activation/KV working set < L2 but
     each forward streams 15 GB of weights (>> 126 MB L2), so L2 is
     implicitly flushed between steps.
  C  `e2e`: the same K steps through the public C ABI with host buffers:
     per step H2D of the token ids + metadata, forward, D2H of the greedy
     first tokens, host wall clock bracketed by device syncs.
Roofline: the dominant kernel (gate/up projection GEMM with fused SiLU*up)
timed live with CUDA events at the dominant step capacity; bytes/flops per
forward from SURVEY.md §8(d).
CPU baseline / `--impl reference`: the CPU forward oracle (oracle/, a port;
the reference itself has no forward — its cost model is closed form) on a
bounded sample, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "prefill req/s and p50/p90 TTFT at 1/2/4/8 B200; HBM GB/s & tensor-pipe % roofline"
UNIT = "req/s"
LAMBDA_PER_MS = 1.0      # saturating offered load per GPU (dispatch sequence for `value`)
DURATION_MS = 4000
LAMBDA_TTFT = 0.25       # sub-saturation load for the reported TTFT p50/p90
DURATION_TTFT_MS = 4000
if os.environ.get("LP_BENCH_QUICK") == "1":  # profiling runs: same phases, short live streams
    DURATION_MS, DURATION_TTFT_MS = 600, 600
TOKEN_SEED = 7


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


def committed_traffic(t_cap: int, n_live: int):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` captures (profiles/r01_dominant_kernel.json),
    if one was taken at this step capacity and live token count; else None."""
    p = ROOT / "profiles" / "r01_dominant_kernel.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    for c in d.get("captures", []):
        if c.get("t_cap") == t_cap and c.get("n_live") == n_live:
            return c.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def gpu_of(local: int) -> int:
    """GPU of this rank. LP_BENCH_SHARE_GPU=1 maps every rank to GPU 0 (a
    functional check of the multi-rank path on a one-GPU box; not a
    measurement)."""
    return 0 if os.environ.get("LP_BENCH_SHARE_GPU") == "1" else local


def dist_init(ws: int, local: int):
    if ws <= 1:
        return None
    import torch
    import torch.distributed as dist
    if os.environ.get("LP_BENCH_SHARE_GPU") == "1":
        dist.init_process_group("gloo")  # NCCL refuses two ranks on one device
        return dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def _reduce(dist, x: float, local: int, op) -> float:
    if dist is None:
        return x
    import torch
    dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{local}"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def dist_max(dist, x: float, local: int) -> float:
    """Timed region of a multi-GPU run = max over ranks (device time)."""
    return _reduce(dist, x, local, dist.ReduceOp.MAX if dist is not None else None)


def dist_sum(dist, x: float, local: int) -> float:
    """Whole-job work = sum over ranks (requests processed)."""
    return _reduce(dist, x, local, dist.ReduceOp.SUM if dist is not None else None)


def aggregate_throughput(dist, reqs: int, dev_ms: float, local: int) -> tuple[float, float, float]:
    """(whole-job req/s, total requests, max-over-ranks ms) for independent
    instances: the job finishes when the slowest rank does."""
    t_max = dist_max(dist, dev_ms, local)
    reqs_all = dist_sum(dist, float(reqs), local)
    return reqs_all / (t_max / 1000.0), reqs_all, t_max


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ workload
def scenario(rank: int, lam: float = LAMBDA_PER_MS, dur: float = DURATION_MS) -> dict:
    from paper_2601_11589_b200 import scenarios as S
    return S.merged(S.SHORT_7B, workload__lambda_per_ms=lam, sim__duration_ms=dur, workload__seed=41 + rank)


def dispatch_sequence(events_log: Path, trace_rows) -> list[dict]:
    by_id = {r.id: r for r in trace_rows}
    out = []
    for line in events_log.read_text().splitlines():
        r = json.loads(line)
        if r["kind"] != "dispatch":
            continue
        ms = []
        for rid in r["reqs"]:
            t = by_id[rid]
            ms.append((rid, t.session, t.L, t.H))
        out.append({"l_pad": r["l_pad"], "depth": r["depth"], "graph": r["graph"], "members": ms})
    return out


def forward_work(model, steps: list[dict]) -> tuple[float, float]:
    """Algorithmic (bytes, flops) of a list of forwards, SURVEY.md §8(d):
    bytes = W + 2*V*h + sum (H+L)*kvB + sum L*h*2 ;
    flops = 2*P*sum L + 4*nq*d*layers*sum L*(H+(L+1)/2) + 2*V*h*n_req."""
    W = model.weight_bytes
    Vh = model.vocab * model.hidden
    kvB = model.kv_bytes_per_token
    P = model.params_nonembed
    byts = flops = 0.0
    for s in steps:
        Ls = [m[2] for m in s["members"]]
        Hs = [m[3] for m in s["members"]]
        byts += W + 2 * Vh + sum((h + l) * kvB for l, h in zip(Ls, Hs)) + sum(Ls) * model.hidden * 2
        flops += (2.0 * P * sum(Ls) + 4.0 * model.n_q_heads * model.head_dim * model.layers *
                  sum(l * (h + (l + 1) / 2) for l, h in zip(Ls, Hs)) + 2.0 * Vh * len(Ls))
    return byts, flops


# ---------------------------------------------------------------- CPU side
class CpuSampler:
    """The CPU oracle forward (torch fp32, all host threads) on a bounded
    sample of the same workload: single-request prefills with L~U[8,255], H=0
    (the config-2 stream), Qwen2.5-7B shape with `layers` of the 28 decoder
    layers + the LM head; the decoder time is scaled to 28 layers (per-layer
    cost is uniform)."""

    def __init__(self, layers: int = 2):
        import torch
        from oracle import forward_oracle as FO
        self.FO = FO
        self.threads = os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        t0 = time.time()
        self.layers = layers
        self.spec = FO.with_layers(FO.QWEN25_7B, layers)
        self.o = FO.OracleModel(self.spec)
        self.setup_s = time.time() - t0
        self.rng = np.random.default_rng(41)
        self.sid = 0

    def sample(self, budget_s: float) -> dict:
        done = 0
        t_layers = t_head = 0.0
        start = time.time()
        while time.time() - start < budget_s or done == 0:
            L = int(self.rng.integers(8, 256))
            toks = self.FO.tokens(TOKEN_SEED, self.sid, 0, L, self.spec.vocab)
            a = time.time()
            self.o.forward([(self.sid, L, 0)], [toks])
            dt = time.time() - a
            b = time.time()
            _ = self.o.lm_head[:1] @ self.o.lm_head.t()  # the LM-head share of one request
            th = time.time() - b
            t_head += th
            t_layers += max(dt - th, 1e-9)
            self.o.kv.pop(self.sid, None)
            self.sid += 1
            done += 1
        per_req = (t_layers * (28 / self.layers) + t_head) / done
        return {"value": 1.0 / per_req, "unit": UNIT, "cores": self.threads, "kind": "port",
                "sample": (f"{done} single-request prefills (L~U[8,255], H=0) of the Qwen2.5-7B-shaped CPU oracle "
                           f"(oracle/forward_oracle.py, torch fp32) with {self.layers}/28 decoder layers + LM head; "
                           f"decoder time scaled x{28 // self.layers}; {time.time() - start:.1f}s sampled "
                           f"(weight synthesis {self.setup_s:.1f}s excluded)")}


def cpu_forward_sample(budget_s: float = 20.0, layers: int = 2) -> dict:
    return CpuSampler(layers).sample(budget_s)


def ref_sim_stats() -> dict | None:
    """The reference simulator (oracle/_ref, compiled from /root/reference) on
    the same config: its CPU cost per dispatch (closed-form forward)."""
    lib = ROOT / "oracle" / "_ref" / "libprefillsim_ref.so"
    if not lib.exists():
        return None
    import ctypes
    from paper_2601_11589_b200 import scenarios as S
    L = ctypes.CDLL(str(lib))
    L.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    secs, nd = ctypes.c_double(), ctypes.c_int64()
    rc = L.ref_simulate(S.text(scenario(0)).encode(), b"", b"", ctypes.byref(secs), ctypes.byref(nd))
    if rc != 0:
        return None
    return {"dispatches": nd.value, "run_s": secs.value, "us_per_dispatch": 1e6 * secs.value / max(1, nd.value)}


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sampler = CpuSampler(layers=2)
    steps_s = []
    per_step = max(0.5, 30.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        r = sampler.sample(budget_s=per_step)
        if i >= args.warmup:
            steps_s.append(r)
    value = float(np.mean([r["value"] for r in steps_s]))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic", "config": {"workload": "c2_short_7b (Qwen2.5-7B-shaped, short-only 8-255, cpu)"},
        "cpu_baseline": {**steps_s[-1], "value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": ref_sim_stats(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
def run_ours(args) -> None:
    ws, rank, local = dist_env()
    dist = dist_init(ws, local)
    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, QWEN25_7B, Member, PrefillInstance
    model = QWEN25_7B
    peaks = load_peaks()

    # Short-only stream: every session is released after its single turn, so a
    # 4096-page pool (262K tokens, 14.7 GB at 7B) is ample and leaves HBM headroom.
    inst = PrefillInstance(model, device=gpu_of(local), max_tokens=16384, max_members=64, kv_pages=4096)
    inst.capture_graphs()  # 6 lengths x 7 depths (GraphGrid defaults)

    # ---- Phase A: live engine run (real GPU service times drive the clock)
    cfg = scenario(rank)
    work = Path(tempfile.mkdtemp(prefix=f"laps_bench_r{rank}_"))
    # Replay mode: the clock is the reference cost model, so the batch
    # composition is exactly the reference scheduler's for this config
    # (deterministic across runs); every dispatch also executes on the GPU.
    st = E.simulate(S.text(cfg), "", work, mode=E.REPLAY, instances=[inst], token_seed=TOKEN_SEED)
    st_ttft = E.simulate(S.text(scenario(rank, LAMBDA_TTFT, DURATION_TTFT_MS)), "", work / "ttft", mode=E.LIVE,
                         instances=[inst], token_seed=TOKEN_SEED)
    E.dump_trace(S.text(cfg), "", work / "trace.txt")
    trace = E.load_trace_dump(work / "trace.txt")
    seq = dispatch_sequence(work / "events.log", trace)
    need = args.warmup + args.steps
    steps = [seq[i % len(seq)] for i in range(need)]

    def members_of(step, uniq):
        return [Member(rid, sid + uniq, L, H) for (rid, sid, L, H) in step["members"]]

    def tokens_of(step):
        return np.concatenate([np.array([E_tok(sid, p) for p in range(H, H + L)], dtype=np.int32)
                               for (_, sid, L, H) in step["members"]])

    from paper_2601_11589_b200.instance import synth_token

    def E_tok(sid, p):
        return synth_token(TOKEN_SEED, sid, p, model.vocab)

    host_tokens = [tokens_of(s) for s in steps]  # host buffers (pinned by the instance on copy)
    kinds = [KIND_GRAPH if s["graph"] else KIND_STANDARD for s in steps]

    # ---- Phase B: timed device throughput
    uniq = 10_000_000
    for i in range(args.warmup):
        inst.submit(steps[i]["l_pad"], steps[i]["depth"], kinds[i], members_of(steps[i], uniq * (i + 1)), host_tokens[i])
        inst.wait()
        for m in steps[i]["members"]:
            inst.release(m[1] + uniq * (i + 1))
    barrier(dist)
    reqs = 0
    launches = 0
    import torch
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects this region
    with ClockSampler(gpu_of(local)) as clk:
        inst.timer_record(0)
        for j in range(args.steps):
            i = args.warmup + j
            ms = members_of(steps[i], uniq * (i + 1))
            inst.submit(steps[i]["l_pad"], steps[i]["depth"], kinds[i], ms, host_tokens[i])
            launches += inst.last_launches()
            for m in ms:
                inst.release(m.session_id)  # stream-ordered reuse of pages
            reqs += len(ms)
        inst.timer_record(1)
        dev_ms = inst.timer_elapsed(0, 1)
    torch.cuda.nvtx.range_pop()
    barrier(dist)
    value, reqs_all, t_max = aggregate_throughput(dist, reqs, dev_ms, local)

    # ---- Phase C: end to end through the C ABI with host buffers
    barrier(dist)
    h2d = d2h = 0
    t0 = time.perf_counter()
    for j in range(args.steps):
        i = args.warmup + j
        ms = members_of(steps[i], uniq * (i + 1) + 1)
        inst.submit(steps[i]["l_pad"], steps[i]["depth"], kinds[i], ms, host_tokens[i])
        inst.wait()
        nt = inst.next_tokens()
        for m in ms:
            inst.release(m.session_id)
        bi, bo = inst.last_io()
        h2d += bi
        d2h += bo
    e2e_s = time.perf_counter() - t0
    e2e_max = dist_max(dist, e2e_s, local)
    e2e_value = reqs_all / e2e_max

    # ---- dominant kernel roofline (gate/up GEMM, fused SiLU*up)
    caps = [s["l_pad"] * s["depth"] if s["graph"] else sum(m[2] for m in s["members"]) for s in steps[args.warmup:]]
    t_cap = int(max(set(caps), key=caps.count))
    live = [sum(m[2] for m in s["members"]) for s, c in zip(steps[args.warmup:], caps) if c == t_cap]
    n_live = int(np.median(live))
    gu_ms = inst.time_gemm(0, 2, t_cap, n_live, iters=20)
    h, I = model.hidden, model.intermediate
    gu_bytes = 2 * I * h * 2 + n_live * h * 2 + n_live * I * 2
    gu_flops = 2.0 * 2 * I * h * n_live
    hbm_bound = gu_bytes / (peaks["hbm_gbs"] * 1e9) > gu_flops / (peaks["bf16_tflops"] * 1e12)
    if hbm_bound:
        achieved, peak, unit = gu_bytes / (gu_ms * 1e-3) / 1e9, peaks["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = gu_flops / (gu_ms * 1e-3) / 1e12, peaks["bf16_tflops"], "TFLOP/s"
    fw_bytes, fw_flops = forward_work(model, steps[args.warmup:])
    ms_per_step = t_max / args.steps

    result = None
    if rank == 0:
        cpu = cpu_forward_sample(budget_s=15.0) if ws == 1 else None
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights from a counter RNG; Poisson short-prefill stream)",
            "config": {"workload": "c2_short_7b: Qwen2.5-7B-shaped, short-only L~U[8,255], 1 turn, "
                                   f"lambda={LAMBDA_PER_MS}/ms/GPU, LAPS temporal instance per GPU, 42 bucket graphs",
                       "model": "qwen2.5-7b-shaped", "parallelism": f"{ws} independent instances (spatial)",
                       "l2": "weights (15 GB/forward) stream through L2 each step; no explicit flush"},
            "ttft_p50_ms": st_ttft.ttft_p50_ms, "ttft_p90_ms": st_ttft.ttft_p90_ms,
            "ttft_load": {"lambda_per_ms": LAMBDA_TTFT, "live_rps": st_ttft.rps, "completed": st_ttft.completed,
                          "slo_violation": st_ttft.slo_violation, "ttft_p99_ms": st_ttft.ttft_p99_ms},
            "saturated_load": {"lambda_per_ms": LAMBDA_PER_MS, "mode": "replay (reference cost-model clock)",
                               "dispatches": st.dispatches, "completed": st.completed,
                               "gpu_forwards": st.gpu_forwards, "gpu_ms_total": st.gpu_ms_total,
                               "gpu_req_per_s": st.completed / (st.gpu_ms_total / 1000.0)},
            "roofline": {"kernel": "gemm_bf16_tn_kernel gate/up (+SiLU*up)", "bound": "hbm" if hbm_bound else "tensor",
                         "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                         "traffic": committed_traffic(t_cap, n_live), "t_cap": t_cap, "n_live": n_live, "avg_ms": gu_ms,
                         "peak_src": peaks["src"],
                         "forward_hbm_gbs": fw_bytes / (t_max * 1e-3) / 1e9 / (1 if ws == 1 else ws),
                         "forward_tflops": fw_flops / (t_max * 1e-3) / 1e12 / (1 if ws == 1 else ws)},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // max(1, args.steps),
                    "d2h_bytes_per_step": d2h // max(1, args.steps)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(result), flush=True)
    inst.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
