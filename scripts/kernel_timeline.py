"""Kernel-level timeline of whole forwards inside the real graphs (diagnostic
build: every forward kernel compiled with -DLP_KTL; block 0 / thread 0 stamps
%globaltimer at entry, after its PDL wait and at exit, see launch.cuh).

For a full-depth forward it prints, per kernel kind, the launches, the mean
time from the PDL wait returning to block 0's exit ("run") and from entry to
the wait returning ("early"), and the boundary cost: how long after block 0
of the previous kernel exited this kernel's wait returned. Block 0 stands in
for its grid (persistent grids and row grids end together within ~1 us).
usage: kernel_timeline.py [--build-only] MODEL [bucket L_PAD DEPTH | chunk H]"""
import ctypes
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402
from paper_2601_11589_b200 import build as B  # noqa: E402

OUT = ROOT / "build" / "ktl"
LIB = OUT / "liblaps_prefill.so"
UNITS = ("ops.cu", "attn.cu", "attn_tc.cu", "gemm_sm100.cu")
KINDS = {1: "gemm", 2: "qkv_post", 3: "resid_rmsnorm", 4: "embed", 5: "attn_warp", 6: "attn_combine",
         7: "attn_tc", 8: "attn_tcp", 9: "gather", 10: "argmax"}


def build():
    B.build()
    OUT.mkdir(parents=True, exist_ok=True)
    objs = []
    for u in UNITS:
        o = OUT / (u + ".o")
        subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, "-DLP_KTL", "-c", str(B.CSRC / u), "-o", str(o)], check=True)
        objs.append(o)
    live = [o for o in sorted(B.BUILD.glob("*.o")) if (B.CSRC / o.name[:-2].replace("__", "/")).exists()]
    objs += [o for o in live if o.name not in {u + ".o" for u in UNITS}]
    cuda_lib = B._cuda_home() / "lib64"
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-L", str(cuda_lib), "-lcudart",
                    "-Xlinker", "-rpath," + str(cuda_lib)], check=True)
    print("built", LIB)


if "--build-only" in sys.argv:
    build()
    sys.exit(0)

import torch  # noqa: E402

N.LIB_PATH = LIB
from paper_2601_11589_b200.instance import KIND_GRAPH, KIND_STANDARD, MODELS, Member, PrefillInstance  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("-")]
name = args[0] if args else "qwen2.5-7b"
mode = args[1] if len(args) > 1 else "bucket"
m = MODELS[name]
L = N.lib()
log = torch.zeros(4 + 4 * 16383, dtype=torch.int64, device="cuda")
for u in ("ops", "attn", "attn_tc", "gemm"):
    f = getattr(L, f"lp_ktl_set_{u}")
    f.argtypes = [ctypes.c_void_p]
    assert f(ctypes.c_void_p(log.data_ptr())) == 0
inst = PrefillInstance(m, max_tokens=8192, max_members=64, kv_pages=1024)
rng = np.random.default_rng(0)
if mode == "bucket":
    lp, dp = int(args[2]), int(args[3])
    inst.capture_graphs(lengths=(lp,), depths=(dp,))
    mem = [Member(i, 100 + i, int(rng.integers(lp // 2 + 1, lp + 1)), 0) for i in range(dp)]
    shape = (lp, dp, KIND_GRAPH)
    title = f"{name} graph {lp}x{dp}"
else:
    H = int(args[2]) if len(args) > 2 else 0
    inst.capture_graphs(lengths=(64,), depths=(1,))
    if H:
        inst.forward(H, 1, KIND_STANDARD, [Member(0, 7, H, 0)], rng.integers(0, m.vocab, H).astype(np.int32))
    mem = [Member(1, 7, 512, H)]
    shape = (512, 1, KIND_STANDARD)
    title = f"{name} 512-token chunk at H={H}"
toks = rng.integers(0, m.vocab, sum(x.new_tokens for x in mem)).astype(np.int32)
for it in range(4):
    if mode == "bucket":
        for x in mem:
            inst.release(x.session_id)
    elif it:
        pass
    log.zero_()
    torch.cuda.synchronize()
    ms = inst.forward(shape[0], shape[1], shape[2], mem, toks)
    if mode != "bucket":
        break  # the chunk's history grows with each forward: time the first one
torch.cuda.synchronize()
n = int(log[0].item())
rec = log[4:4 + 4 * n].view(n, 4).cpu().numpy().astype(np.int64)
rec = rec[np.argsort(rec[:, 1])]
kinds = rec[:, 0] >> 32
meta = rec[:, 0] & 0xFFFFFFFF
t0 = rec[:, 1].min()
entry, start, end = (rec[:, 1] - t0) / 1e3, (rec[:, 2] - t0) / 1e3, (rec[:, 3] - t0) / 1e3
start = np.where(rec[:, 2] >= rec[:, 1], start, entry)  # no wait stamp seen: count from entry
print(f"== {title}: forward {ms:.3f} ms (events), {n} kernels, span {end.max():.1f} us")
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i in range(n):
    k = KINDS.get(int(kinds[i]), str(kinds[i]))
    if k == "gemm":
        k = f"gemm M={int(meta[i])}"
    a = agg[k]
    a[0] += 1
    a[1] += end[i] - start[i]
    a[2] += start[i] - entry[i]
    a[3] += (start[i] - end[i - 1]) if i else 0.0
tot_run = sum(v[1] for v in agg.values())
tot_gap = sum(v[3] for v in agg.values())
for k, (c, run, early, gap) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:22s} n={c:4d}  run {run / c:8.2f} us  early {early / c:7.2f} us  boundary {gap / c:6.2f} us  "
          f"(run total {run / 1e3:7.3f} ms, boundary total {gap / 1e3:6.3f} ms)")
print(f"  sum of runs {tot_run / 1e3:.3f} ms, sum of boundaries {tot_gap / 1e3:.3f} ms (negative = overlap)")
inst.close()
