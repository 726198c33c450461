"""Run one GEMM config a few times (for ncu). usage: gemm_one.py M N K mode bn pair splits iters"""
import ctypes, sys
import torch
sys.path.insert(0, '.')
from paper_2601_11589_b200 import _native as N
M, Nt, K, mode, bn, pair, splits, iters = map(int, sys.argv[1:9])
L = N.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
W = (torch.randn(M, K, device='cuda') * 0.05).bfloat16(); X = torch.randn(Nt, K, device='cuda').bfloat16()
out = torch.empty(Nt, M, device='cuda', dtype=torch.float32)
ws = torch.empty(splits, Nt, M, device='cuda', dtype=torch.float32)
ldo = M // 2 if mode == 2 else M
ts = []
for i in range(iters):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    N.check(L.lpk_gemm(P(W), P(X), P(out), P(ws), None, M, Nt, K, splits, mode, bn, ldo, None, None, pair))
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
t = sorted(ts)[len(ts) // 2]
print(f"M={M} N={Nt} K={K} mode={mode} bn={bn} pair={pair}: {t*1e3:.1f} us  {2.0*M*Nt*K/t/1e9:.0f} TF/s")
