#!/usr/bin/env python3
"""Benchmark: LAPS prefill tier on B200 (BASELINE.json metric "prefill req/s
and p50/p90 TTFT at 1/2/4/8 B200; HBM GB/s & tensor-pipe % roofline").

Workload = BASELINE.json config 4 — the configuration the metric is quoted on
(BASELINE.md §4): Qwen2.5-32B-shaped random-init bf16 decoder, mixed LMsys-like
stream (short 8-255 / long 1025-4096 new tokens, 63% short first turns, 81%
later, 1-6 turns per session, seed 7), the 42 length-bucket CUDA graphs plus
512-token chunk graphs, one LAPS temporal instance at N = 1. At N > 1 the same
stream at N x the arrival rate is served by N GPUs in spatial disaggregation
behind the length-aware router (ceil(N/2) short-pool GPUs), all driven by ONE
host engine (the reference's router is global, sim.cpp:379-411), so
"scaling": "weak" (per-GPU load fixed).

A step = one dispatched batch forward of the reference scheduler per GPU (a
graph bucket replay or a long-prompt chunk): the window holds K x N dispatches
at N GPUs, so every GPU runs ~K forwards (weak scaling). The engine runs in REPLAY mode: its
clock is the reference cost model, so the dispatch sequence is exactly the
reference scheduler's (deterministic), and every dispatch executes on its GPU
asynchronously (N GPUs concurrently). Dispatches [0, W) warm up (and build the
sessions' KV), [W, W + K) are the timed window:
  value  requests per second of device time: requests finished in the window
         / max over GPUs of the CUDA-event time around the window's forwards
         (GPUs idle at the start). A long prompt's chunk counts 1/chunks of a
         request, so a window boundary cutting a chunk chain does not bias it.
  e2e    the same window on host steady_clock through the public C ABI
         (lp_sim_run_ex -> lp_submit_async): token ids synthesized and copied
         H2D from host memory each step, forwards, first tokens copied D2H and
         read by the host, engine time included.
TTFT p50/p90: a WALL-clock run (arrivals released in real time, completions
from CUDA events) at a sub-saturating rate.
Roofline: the dominant kernel (the gate/up GEMM of a full 512-token chunk,
~half of a chunk forward) timed live with CUDA events on the instance stream;
DRAM traffic from the committed `ncu --set full` capture of the same launch.
CPU baseline / --impl reference: the CPU forward oracle (oracle/, a port — the
reference's own "forward" is a closed form with no logits) over the window's
dispatches, one decoder layer of the 32B shape timed and scaled x64, plus the
LM head, all host threads.
"""
from __future__ import annotations

import argparse
import csv
import json
import math
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
TOKEN_SEED = 7
LAMBDA_PER_GPU = 0.02      # req/ms offered per GPU (the reference cost model is saturated)
DURATION_MS = 60000        # of the replayed stream (only W + K dispatches execute on the GPU)
LAMBDA_TTFT_PER_GPU = 0.008
DURATION_TTFT_MS = 8000
DOMINANT = {"which": 2, "t_cap": 512, "n_live": 512}  # gate/up GEMM (+SiLU*up) of a full C_l chunk


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "src": "fallback (B200_PROFILING.md)"}


def committed_traffic(model_name: str, which: int, t_cap: int, n_live: int):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/r02_dominant_kernel.json)."""
    p = ROOT / "profiles" / "r02_dominant_kernel.json"
    if not p.exists():
        return None
    for c in reversed(json.loads(p.read_text()).get("captures", [])):  # the latest capture of that launch
        if (c.get("model"), c.get("which"), c.get("t_cap"), c.get("n_live")) == (model_name, which, t_cap, n_live):
            return c.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = sorted(set(devices))
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        ids = ",".join(str(d) for d in self.devices)
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={ids}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        ok = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in ok if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in ok if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in ok for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(ok)}


# --------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    return ws, rank


def dist_init(ws: int):
    """Under torchrun, rank 0 drives every GPU from one host engine (the
    reference's router is one global component); the other ranks only join
    the barriers (gloo, no GPU work)."""
    if ws <= 1:
        return None
    import torch.distributed as dist
    dist.init_process_group("gloo")
    return dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ workload
def scenario(n_gpus: int, lam_per_gpu: float, duration_ms: float) -> dict:
    from paper_2601_11589_b200 import scenarios as S
    over = {"workload__lambda_per_ms": lam_per_gpu * n_gpus, "sim__duration_ms": duration_ms}
    if n_gpus > 1:
        # Spatial pools start at the reference's default split (ceil(N/2) short) and
        # the Alg. 2 controller moves GPUs between pools (as in config 5).
        over.update(sim__disagg="spatial", sim__instances=n_gpus, sim__initial_short_instances=(n_gpus + 1) // 2,
                    sim__controller="true" if n_gpus > 2 else "false")
    return S.merged(S.LMSYS_32B, **over)


def window_dispatches(events_log: Path, first: int, count: int) -> list[dict]:
    """Dispatch records [first, first + count) of an events.log (the GPU
    dispatch index equals the dispatch record index)."""
    out = []
    k = 0
    for line in events_log.read_text().splitlines():
        r = json.loads(line)
        if r["kind"] != "dispatch":
            continue
        if first <= k < first + count:
            out.append(r)
        k += 1
    return out


def request_equivalents(disp: list[dict]) -> float:
    """Requests finished by these dispatches, a long prompt's chunk counting
    1/chunks of its request (every chunk of a k-chunk prompt is 1/k)."""
    n = 0.0
    for r in disp:
        if r["reason"] == "long_chunk":
            n += 1.0 / r["chunks"]
        else:
            n += len(r["reqs"])
    return n


def member_rows(disp: list[dict], trace) -> list[list[tuple[int, int, int]]]:
    """(session, L, H) of every member of every dispatch (chunk histories
    accumulated as in scheduler.cpp:322-338)."""
    by = {t.id: t for t in trace}
    out = []
    for r in disp:
        rows = []
        for q in r["reqs"]:
            t = by[q]
            if r["reason"] == "long_chunk":
                rows.append((t.session, r["real"], t.H + (r["chunk"] - 1) * 512))
            else:
                rows.append((t.session, t.L, t.H))
        out.append(rows)
    return out


# ---------------------------------------------------------------- CPU side
class CpuSampler:
    """The CPU forward oracle (torch fp32, all host threads) on the window's
    dispatches: one decoder layer of the Qwen2.5-32B shape + the LM head per
    member; the layer time is scaled x64 (per-layer cost is uniform). History
    KV is a placeholder of the right shape (attention cost depends on the
    history length, not its values)."""

    LAYERS = 1

    def __init__(self):
        import torch
        from oracle import forward_oracle as FO
        self.FO, self.torch = FO, torch
        self.threads = os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        t0 = time.time()
        self.spec = FO.with_layers(FO.QWEN25_32B, self.LAYERS)
        self.o = FO.OracleModel(self.spec)
        self.setup_s = time.time() - t0

    def step(self, rows) -> float:
        """Scaled CPU seconds of one dispatch."""
        torch, s = self.torch, self.spec
        members, toks = [], []
        for i, (sid, L, H) in enumerate(rows):
            key = 10_000_000 + i
            z = torch.zeros(H, s.n_kv_heads, s.head_dim)
            self.o.kv[key] = [[z, z.clone()] for _ in range(s.layers)]
            members.append((key, L, H))
            toks.append(self.FO.tokens(TOKEN_SEED, sid, H, L, s.vocab))
        t0 = time.time()
        self.o.forward(members, toks)
        dt = time.time() - t0
        th0 = time.time()
        _ = self.o.lm_head[: len(rows)] @ self.o.lm_head.t()  # the LM-head share
        th = time.time() - th0
        for key, _, _ in members:
            self.o.kv.pop(key, None)
        return max(dt - th, 1e-9) * (64 / self.LAYERS) + th

    def run(self, disp, rows, budget_s: float) -> dict:
        t_cpu = reqs = 0.0
        done = 0
        start = time.time()
        for r, rw in zip(disp, rows):
            t_cpu += self.step(rw)
            reqs += request_equivalents([r])
            done += 1
            if time.time() - start > budget_s:
                break
        return {"value": reqs / t_cpu, "unit": UNIT, "cores": self.threads, "kind": "port",
                "sample": (f"{done} of the window's dispatches (same members, L and H) through the CPU oracle "
                           f"(oracle/forward_oracle.py, torch fp32): 1 of 64 decoder layers of the Qwen2.5-32B "
                           f"shape timed and scaled x64, + LM head; {reqs:.2f} request-equivalents in "
                           f"{t_cpu:.1f} scaled CPU-s ({time.time() - start:.1f}s sampled, weight synthesis "
                           f"{self.setup_s:.1f}s excluded)")}


def cost_model_window(n_gpus: int, first: int, count: int):
    """The reference scheduler's dispatch sequence (cost-model clock) and
    the trace, without a GPU."""
    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    cfg = scenario(n_gpus, LAMBDA_PER_GPU, DURATION_MS)
    d = Path(tempfile.mkdtemp(prefix="laps_bench_cm_"))
    E.simulate(S.text(cfg), "", d, mode=E.COST_MODEL)
    E.dump_trace(S.text(cfg), "", d / "trace.txt")
    trace = E.load_trace_dump(d / "trace.txt")
    return window_dispatches(d / "events.log", first, count), trace


def ref_sim_stats(cfg: dict) -> dict | None:
    """The reference simulator (oracle/_ref, compiled from /root/reference):
    its CPU cost per dispatch (closed-form forward), same config."""
    lib = ROOT / "oracle" / "_ref" / "libprefillsim_ref.so"
    if not lib.exists():
        return None
    import ctypes
    from paper_2601_11589_b200 import scenarios as S
    L = ctypes.CDLL(str(lib))
    L.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    secs, nd = ctypes.c_double(), ctypes.c_int64()
    if L.ref_simulate(S.text(cfg).encode(), b"", b"", ctypes.byref(secs), ctypes.byref(nd)) != 0:
        return None
    return {"dispatches": nd.value, "run_s": secs.value, "us_per_dispatch": 1e6 * secs.value / max(1, nd.value)}


def workload_label(n: int) -> str:
    mode = "1 LAPS temporal instance" if n == 1 else f"{n} GPUs spatial ({(n + 1) // 2} short-pool) behind one router"
    return (f"c4_lmsys_32b: Qwen2.5-32B-shaped, mixed LMsys-like (short 8-255 63%/81%, long 1025-4096, 1-6 turns, "
            f"seed 7), lambda={LAMBDA_PER_GPU * n:g}/ms, {mode}, 42 bucket graphs + 512-token chunk graphs")


def run_reference(args) -> None:
    ws, rank = dist_env()
    if rank != 0:
        return
    disp, trace = cost_model_window(args.gpus, args.warmup * args.gpus, args.steps * args.gpus)
    rows = member_rows(disp, trace)
    sampler = CpuSampler()
    # One step = one window dispatch (bounded: ~3 s of CPU work each at most).
    t_cpu = reqs = 0.0
    n = 0
    t0 = time.time()
    for r, rw in zip(disp, rows):
        if time.time() - t0 > 150:
            break
        t_cpu += sampler.step(rw)
        reqs += request_equivalents([r])
        n += 1
    value = reqs / t_cpu
    sample = (f"{n} of the {len(disp)} window dispatches (the same members, L and H as the GPU arm) through the "
              f"CPU oracle (torch fp32, {sampler.threads} threads): 1 of 64 decoder layers of the Qwen2.5-32B shape "
              f"timed and scaled x64, + LM head; request-equivalents {reqs:.2f} in {t_cpu:.1f} scaled CPU-s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_cpu / max(1, n),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (random-init weights from a counter RNG; Poisson LMsys-like stream)",
        "config": {"workload": workload_label(args.gpus)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": sampler.threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": ref_sim_stats(scenario(args.gpus, LAMBDA_PER_GPU, DURATION_MS)),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
def forward_work(model, rows) -> tuple[float, float]:
    """Algorithmic (bytes, flops) of one forward from forwards.csv fields
    (SURVEY.md §8(d)): bytes = W + 2*V*h + (T + sum H)*kvB + T*h*2;
    flops = 2*P*T + 4*nq*d*layers*pairs + 2*V*h*n_req."""
    Vh = model.vocab * model.hidden
    T, Hs, pairs, n = int(rows["tokens"]), int(rows["hist_tokens"]), float(rows["attn_pairs"]), int(rows["members"])
    b = model.weight_bytes + 2 * Vh + (T + Hs) * model.kv_bytes_per_token + T * model.hidden * 2
    f = 2.0 * model.params_nonembed * T + 4.0 * model.n_q_heads * model.head_dim * model.layers * pairs + 2.0 * Vh * n
    return b, f


def run_ours(args) -> None:
    ws, rank = dist_env()
    dist = dist_init(ws)
    if rank != 0:  # rank 0 drives every GPU (one router); the others only sync
        barrier(dist)
        barrier(dist)
        dist.destroy_process_group()
        return
    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    from paper_2601_11589_b200.instance import MODELS, PrefillInstance
    n = args.gpus
    model_name = os.environ.get("LP_BENCH_MODEL", "qwen2.5-32b")
    model = MODELS[model_name]
    share = os.environ.get("LP_BENCH_SHARE_GPU") == "1"  # functional check of N>1 on a 1-GPU box
    devices = [0 if share else i for i in range(n)]
    peaks = load_peaks()
    t_setup = time.time()
    insts = [PrefillInstance(model, device=dev, max_tokens=16384, max_members=64,
                             kv_pages=(4096 // n if share else 0)) for dev in devices]
    for inst in insts:
        inst.capture_graphs()
    setup_s = time.time() - t_setup

    cfg = scenario(n, LAMBDA_PER_GPU, DURATION_MS)
    work = Path(tempfile.mkdtemp(prefix="laps_bench_"))
    barrier(dist)
    with ClockSampler(devices) as clk:
        st = E.simulate(S.text(cfg), "", work / "replay", mode=E.REPLAY, instances=insts, token_seed=TOKEN_SEED,
                        window=(args.warmup * n, args.steps * n), stop_after_window=True)
    if st.window_dispatches != args.steps * n:
        raise RuntimeError(f"window ran {st.window_dispatches} dispatches, expected {args.steps}")
    disp = window_dispatches(work / "replay" / "events.log", args.warmup * n, args.steps * n)
    reqs = request_equivalents(disp)
    value = reqs / (st.window_device_ms / 1000.0)
    e2e_value = reqs / (st.window_wall_ms / 1000.0)

    # Per-forward roofline over the window's forwards (forwards.csv).
    fw = [r for r in csv.DictReader(open(work / "replay" / "forwards.csv")) if r["window"] == "1"]
    fb = ff = floor = gpu_sum = 0.0
    for r in fw:
        b, f = forward_work(model, r)
        fb += b
        ff += f
        floor += max(b / (peaks["hbm_gbs"] * 1e9), f / (peaks["bf16_tflops_sustained"] * 1e12))
        gpu_sum += float(r["gpu_ms"]) * 1e-3
    kinds = {"graph": sum(1 for r in fw if r["graph"] == "1"),
             "chunk_or_standard": sum(1 for r in fw if r["graph"] == "0")}

    # TTFT: wall clock, arrivals in real time, completions from CUDA events.
    cfg_ttft = scenario(n, LAMBDA_TTFT_PER_GPU, DURATION_TTFT_MS)
    live = E.simulate(S.text(cfg_ttft), "", work / "wall", mode=E.WALL, instances=insts, token_seed=TOKEN_SEED)
    # The same stream on the virtual clock advanced by each measured forward
    # (LIVE mode): TTFT from device service times alone, no host costs.
    virt = E.simulate(S.text(cfg_ttft), "", work / "live", mode=E.LIVE, instances=insts, token_seed=TOKEN_SEED)

    # Dominant kernel: gate/up GEMM of a full 512-token chunk, CUDA events.
    dk = DOMINANT
    gu_ms = insts[0].time_gemm(0, dk["which"], dk["t_cap"], dk["n_live"], iters=20)
    h, I = model.hidden, model.intermediate
    gu_flops = 2.0 * 2 * I * h * dk["n_live"]
    gu_bytes = 2 * I * h * 2 + dk["n_live"] * h * 2 + dk["n_live"] * I * 2
    tensor = gu_flops / (peaks["bf16_tflops"] * 1e12) >= gu_bytes / (peaks["hbm_gbs"] * 1e9)
    achieved = gu_flops / (gu_ms * 1e-3) / 1e12 if tensor else gu_bytes / (gu_ms * 1e-3) / 1e9
    peak = peaks["bf16_tflops"] if tensor else peaks["hbm_gbs"]

    cpu = None
    if n == 1:
        trace_path = work / "trace.txt"
        E.dump_trace(S.text(cfg), "", trace_path)
        cpu = CpuSampler().run(disp, member_rows(disp, E.load_trace_dump(trace_path)), budget_s=20.0)

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": st.window_device_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights from a counter RNG; Poisson LMsys-like multi-turn stream)",
        "config": {"workload": workload_label(n), "model": f"{model_name}-shaped",
                   "parallelism": "1 temporal instance" if n == 1 else f"{n} instances, spatial, one router",
                   "step": "one dispatch of the reference scheduler per GPU (window = steps x n_gpus dispatches, "
                           "REPLAY clock); requests = request-equivalents "
                           "(a chunk of a k-chunk long prompt counts 1/k)",
                   "l2": "no explicit flush: every forward streams the 62 GB of 32B weights (>> 126 MB L2)",
                   "shared_gpu": share},
        "requests_in_window": reqs,
        "window": {"dispatches": st.window_dispatches, "graph_forwards": kinds["graph"],
                   "chunk_or_standard_forwards": kinds["chunk_or_standard"], "history_fills": st.window_fills,
                   "device_ms": st.window_device_ms, "wall_ms": st.window_wall_ms,
                   "forward_hbm_gbs": fb / gpu_sum / 1e9 if gpu_sum else None,
                   "forward_tflops": ff / gpu_sum / 1e12 if gpu_sum else None,
                   "forward_roofline_frac": floor / gpu_sum if gpu_sum else None},
        "ttft_p50_ms": live.ttft_p50_ms, "ttft_p90_ms": live.ttft_p90_ms,
        "ttft_run": {"clock": "wall (steady_clock; arrivals released in real time; completions = CUDA events)",
                     "lambda_per_ms": LAMBDA_TTFT_PER_GPU * n, "duration_ms": DURATION_TTFT_MS,
                     "completed": live.completed, "rps": live.rps, "slo_violation": live.slo_violation,
                     "ttft_p99_ms": live.ttft_p99_ms, "engine_wall_s": live.engine_wall_s,
                     "kv_migrations": live.kv_migrations,
                     "measured_service_clock": {"ttft_p50_ms": virt.ttft_p50_ms, "ttft_p90_ms": virt.ttft_p90_ms,
                                                "note": "LIVE mode: virtual clock advanced by each forward's "
                                                        "CUDA-event time (no engine / H2D / launch cost)"}},
        "roofline": {"kernel": "gemm_bf16_tn_kernel gate/up (+SiLU*up), 32B, full 512-token chunk",
                     "bound": "tensor" if tensor else "hbm", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s" if tensor else "GB/s", "frac": achieved / peak,
                     "traffic": committed_traffic(model_name, dk["which"], dk["t_cap"], dk["n_live"]),
                     "algorithmic_bytes": gu_bytes, "algorithmic_flops": gu_flops, "avg_ms": gu_ms,
                     "peak_src": peaks["src"] + " burst (kernel timed alone)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": st.window_h2d_bytes // max(1, args.steps),
                "d2h_bytes_per_step": st.window_d2h_bytes // max(1, args.steps)},
        "gpu_launches": st.window_kernels,
        "clocks": clk.summary(),
        "setup_s": setup_s,
    }
    if n == 1 and not share and os.environ.get("LP_BENCH_C2", "1") == "1":
        for inst in insts:
            inst.close()
        insts = []
        result["extra_configs"] = {"c2_short_7b": run_c2(args)}
    print(json.dumps(result), flush=True)
    if os.environ.get("LP_BENCH_OUT"):  # keep events.log / forwards.csv of the run (profiling)
        import shutil
        shutil.copytree(work, os.environ["LP_BENCH_OUT"], dirs_exist_ok=True)
    for inst in insts:
        inst.close()
    barrier(dist)
    if dist is not None:
        dist.destroy_process_group()


def run_c2(args) -> dict:
    """BASELINE config 2 as an extra key (round-1 headline): Qwen2.5-7B-shaped,
    short-only stream (8-255 tokens, 1 turn, 1 req/ms: the reference
    scheduler batches deep), one temporal instance; same window method."""
    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    from paper_2601_11589_b200.instance import QWEN25_7B, PrefillInstance
    inst = PrefillInstance(QWEN25_7B, device=0, max_tokens=16384, max_members=64, kv_pages=4096)
    inst.capture_graphs()
    cfg = S.merged(S.SHORT_7B, workload__lambda_per_ms=1.0, sim__duration_ms=4000)
    work = Path(tempfile.mkdtemp(prefix="laps_bench_c2_"))
    st = E.simulate(S.text(cfg), "", work / "replay", mode=E.REPLAY, instances=[inst], token_seed=TOKEN_SEED,
                    window=(args.warmup, args.steps), stop_after_window=True)
    reqs = request_equivalents(window_dispatches(work / "replay" / "events.log", args.warmup, args.steps))
    cfg_t = S.merged(S.SHORT_7B, workload__lambda_per_ms=0.25, sim__duration_ms=4000)
    wall = E.simulate(S.text(cfg_t), "", work / "wall", mode=E.WALL, instances=[inst], token_seed=TOKEN_SEED)
    inst.close()
    return {"workload": "Qwen2.5-7B-shaped, short-only L~U[8,255], 1 turn, lambda=1.0/ms, 1 temporal instance, "
                        "42 bucket graphs", "steps": args.steps,
            "value": reqs / (st.window_device_ms / 1000.0), "unit": UNIT,
            "e2e": reqs / (st.window_wall_ms / 1000.0), "ms_per_step": st.window_device_ms / args.steps,
            "gpu_launches": st.window_kernels, "ttft_p50_ms": wall.ttft_p50_ms, "ttft_p90_ms": wall.ttft_p90_ms,
            "ttft_clock": "wall, lambda=0.25/ms"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
