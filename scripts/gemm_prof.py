"""Per-CTA phase timeline of the tcgen05 GEMM inside real forwards
(diagnostic build: gemm_sm100.cu under -DLP_GEMM_PROF, %globaltimer stamps).

Builds build/prof/liblaps_prefill.so, loads it instead of the product
library, runs one decoder layer of MODEL on (a) a 512-token chunk (chunk
graph) and (b) a 256x1 graph bucket with 200 tokens, and for each projection
prints, relative to the earliest CTA entry of that launch (us): CTA entry
spread, setup (barriers + TMEM + cluster sync), the predecessor wait (PDL),
first operands landed, the MMA span, the epilogue tail, and the end.
usage: gemm_prof.py [--build-only] [MODEL]"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402
from paper_2601_11589_b200 import build as B  # noqa: E402

PROF = ROOT / "build" / "prof_gemm"
LIB = PROF / "liblaps_prefill.so"


def build_prof():
    B.build()
    PROF.mkdir(parents=True, exist_ok=True)
    obj = PROF / "gemm_sm100.o"
    src = B.CSRC / "gemm_sm100.cu"
    subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, "-DLP_GEMM_PROF", "-c", str(src), "-o", str(obj)], check=True)
    live = [o for o in sorted(B.BUILD.glob("*.o")) if (B.CSRC / o.name[:-2].replace("__", "/")).exists()]
    objs = [o for o in live if o.name != "gemm_sm100.cu.o"] + [obj]
    cuda_lib = B._cuda_home() / "lib64"
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-L", str(cuda_lib), "-lcudart",
                    "-Xlinker", "-rpath," + str(cuda_lib)], check=True)
    print("built", LIB)


if "--build-only" in sys.argv:
    build_prof()
    sys.exit(0)

N.LIB_PATH = LIB
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

L = N.lib()
L.lp_debug_gemm_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
CTAS, EV = 160, 12
buf = np.zeros((CTAS, EV), dtype=np.uint64)
name = next((a for a in sys.argv[1:] if not a.startswith("-")), "qwen2.5-32b")
m = MODELS[name].with_layers(int(os.environ.get("LP_PROF_LAYERS", "1")))
inst = PrefillInstance(m, max_tokens=4096, max_members=32, kv_pages=512)
inst.capture_graphs(lengths=(16, 256), depths=(1,))
rng = np.random.default_rng(0)
qkv_out = (m.n_q_heads + 2 * m.n_kv_heads) * m.head_dim
proj = {"qkv": (qkv_out, m.hidden), "o": (m.hidden, m.n_q_heads * m.head_dim),
        "gate_up": (2 * m.intermediate, m.hidden), "down": (m.hidden, m.intermediate)}


def scenario(title, l_pad, kind, n_tok):
    print(f"== {name} {title}")
    for pname, (M, K) in proj.items():
        sid = 1000
        L.lp_debug_gemm_prof(None, 0, M, K)
        for _ in range(3):
            inst.release(sid)
            ms = inst.forward(l_pad, 1, kind, [Member(0, sid, n_tok, 0)], rng.integers(0, m.vocab, n_tok).astype(np.int32))
        L.lp_debug_gemm_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size, 0, 0)
        b = buf.astype(np.int64)
        used = np.nonzero(b[:, 0])[0]
        if len(used) == 0:
            print(f"  {pname}: no launch recorded")
            continue
        t0 = b[used, 0].min()
        rel = (b[used] - t0) / 1e3
        lead = [i for i, c in enumerate(used) if b[c, 4] != 0]

        def med(x):
            return float(np.median(x)) if len(x) else float("nan")
        print(f"  {pname:8s} M={M} K={K}: forward {ms:.3f} ms, {len(used)} CTAs, units/CTA {med(b[used, 9]):.0f} | "
              f"entry med/max {med(rel[:, 0]):.2f}/{rel[:, 0].max():.2f} | setup {med(rel[:, 1] - rel[:, 0]):.2f} | "
              f"pdl_wait returns {med(rel[:, 2]):.2f} (max {rel[:, 2].max():.2f}) | first operands +{med(rel[lead, 4] - rel[lead, 2]):.2f} | "
              f"MMA span {med(rel[lead, 5] - rel[lead, 4]):.2f} (max {np.max(rel[lead, 5] - rel[lead, 4]):.2f}) | "
              f"last acc -> epi done {med(rel[:, 7] - rel[:, 8]):.2f} (clk: tmem ld {med(b[used, 10]):.0f}, rest {med(b[used, 11]):.0f}) | end med/max {med(rel[:, 7]):.2f}/{rel[:, 7].max():.2f} us",
              flush=True)


only = os.environ.get("LP_PROF_ONLY", "")
if only in ("", "chunk"):
    scenario("512-token chunk (chunk graph)", 512, KIND_STANDARD, 512)
if only in ("", "bucket"):
    scenario("256x1 graph bucket, 200 tokens", 256, KIND_GRAPH, 200)
if only in ("", "small"):
    scenario("16x1 graph bucket, 12 tokens", 16, KIND_GRAPH, 12)
inst.close()
