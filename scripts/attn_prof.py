"""Per-step timeline of the tcgen05 attention kernel (diagnostic build).

Builds build/prof/liblaps_prefill.so with attn_tc.cu compiled under
-DLP_ATTN_PROF (clock64 stamps: MMA issuer, one softmax warp, K producer) and
the other objects of the normal build, loads it instead of the product
library, runs one Qwen2.5-7B layer on (a) a 512-token chunk at history H and
(b) 16 members x 16 tokens at H=1024 (eager standard batch), and prints the
median per-step intervals over the instrumented CTAs.
usage: attn_prof.py [--build-only] [H]"""
import ctypes
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402
from paper_2601_11589_b200 import build as B  # noqa: E402

PROF = ROOT / "build" / "prof"
LIB = PROF / "liblaps_prefill.so"


def build_prof():
    B.build()
    PROF.mkdir(parents=True, exist_ok=True)
    obj = PROF / "attn_tc.o"
    src = B.CSRC / "attn_tc.cu"
    subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, "-DLP_ATTN_PROF", "-c", str(src), "-o", str(obj)], check=True)
    live = [o for o in sorted(B.BUILD.glob("*.o")) if (B.CSRC / o.name[:-2].replace("__", "/")).exists()]
    objs = [o for o in live if o.name != "attn_tc.cu.o"] + [obj]
    cuda_lib = B._cuda_home() / "lib64"
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-L", str(cuda_lib), "-lcudart",
                    "-Xlinker", "-rpath," + str(cuda_lib)], check=True)
    print("built", LIB, [o.name for o in objs])


if "--build-only" in sys.argv:
    build_prof()
    sys.exit(0)

N.LIB_PATH = LIB
from paper_2601_11589_b200.instance import KIND_STANDARD, QWEN25_7B, Member, PrefillInstance  # noqa: E402

L = N.lib()
L.lp_debug_attn_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_size_t]
CTAS, STEPS = 128, 64
buf = np.zeros((CTAS, 3, STEPS, 8), dtype=np.uint64)

m = QWEN25_7B.with_layers(1)
inst = PrefillInstance(m, max_tokens=4096, max_members=32, kv_pages=1024, use_graphs=False)
rng = np.random.default_rng(0)
sid = [100]


def fill(s, H):
    for p in range(0, H, 4096):
        n = min(4096, H - p)
        inst.forward(n, 1, KIND_STANDARD, [Member(0, s, n, p)], rng.integers(0, m.vocab, n).astype(np.int32))


def run(title, members_spec):
    ms = []
    for i, (Lq, H) in enumerate(members_spec):
        s = sid[0]
        sid[0] += 1
        fill(s, H)
        ms.append(Member(i, s, Lq, H))
    toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in ms)).astype(np.int32)
    lp = max(x.new_tokens for x in ms)
    for _ in range(2):
        L.lp_debug_attn_prof_reset()
        t = inst.forward(lp, len(ms), KIND_STANDARD, ms, toks)
    L.lp_debug_attn_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
    for x in ms:
        inst.release(x.session_id)
    b = buf.astype(np.int64)
    used = [c for c in range(CTAS) if b[c, 0, 0, 0] != 0]
    print(f"== {title}: forward {t:.3f} ms, {len(used)} instrumented CTAs (KV head 0)")
    rows = []
    for c in used:
        mma, sm, prod = b[c, 0], b[c, 1], b[c, 2]
        n = int(np.count_nonzero(mma[:, 0]))
        if n < 3:
            continue
        step = np.diff(mma[:n, 1])                       # p_ready(s) -> p_ready(s+1)
        rows.append(dict(
            n=n,
            step=np.median(step),
            mma_wait_p=np.median(mma[1:n, 1] - mma[1:n, 0]),
            mma_wait_v=np.median(mma[1:n, 2] - mma[1:n, 1]),
            mma_issue=np.median(mma[1:n, 3] - mma[1:n, 2]),
            sm_wait_s=np.median(sm[1:n, 1] - sm[1:n, 0]),
            sm_exp=np.median(sm[1:n, 2] - sm[1:n, 1]),
            sm_ldtm=np.median(sm[1:n, 4] - sm[1:n, 1]),
            sm_xchg=np.median(sm[1:n, 5] - sm[1:n, 4]),
            sm_exps=np.median(sm[1:n, 2] - sm[1:n, 5]),
            sm_pfree=np.median(sm[1:n, 6] - sm[1:n, 2]),
            sm_pstore=np.median(sm[1:n, 3] - sm[1:n, 6]),
            sm_tail=np.median(sm[1:n, 3] - sm[1:n, 2]),
            prod_wait=np.median(prod[2:n, 1] - prod[2:n, 0]) if n > 3 else 0,
            first=int(sm[0, 1] - prod[0, 1]) if prod[0, 1] else 0,
        ))
    if not rows:
        print("no multi-step CTAs")
        return
    keys = list(rows[0])
    med = {k: float(np.median([r[k] for r in rows])) for k in keys}
    print("  median over CTAs (cycles): " + ", ".join(f"{k}={med[k]:.0f}" for k in keys))


H = int(sys.argv[1]) if len(sys.argv) > 1 else 3584
run(f"512-token chunk, H={H}", [(512, H)])
run("16 members x 16 tokens, H=1024", [(16, 1024)] * 16)
inst.close()
