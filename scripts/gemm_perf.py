"""GEMM micro-benchmark (weight-streaming and compute-bound shapes)."""
import ctypes, json, sys
import torch
sys.path.insert(0, '.')
from paper_2601_11589_b200 import _native as N
L = N.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
peaks = json.load(open('MEASURED_PEAKS.json')) if __import__('os').path.exists('MEASURED_PEAKS.json') else {"hbm_gbs": 6545.6, "bf16_tflops": 1664.4}
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
def bench(M, Nt, K, splits, mode, bn, iters=20, pair=1):
    W = torch.randn(M, K, device='cuda').bfloat16(); X = torch.randn(Nt, K, device='cuda').bfloat16()
    out = torch.empty(Nt, M, device='cuda', dtype=torch.bfloat16)
    ws = torch.empty(splits, Nt, M, device='cuda', dtype=torch.float32) if mode == 1 else None
    ldo = M // 2 if mode == 2 else M
    def run(): N.check(L.lpk_gemm(P(W), P(X), P(out), P(ws), None, M, Nt, K, splits, mode, bn, ldo, None, None, pair))
    for _ in range(3): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts)//2] * 1e-3
    byts = M * K * 2 + Nt * K * 2 + Nt * M * (4 * splits if mode == 1 else 2)
    fl = 2.0 * M * Nt * K
    print(f"M={M:6d} N={Nt:5d} K={K:5d} s={splits} bn={bn:3d} p={pair} mode={mode}: {t*1e6:8.1f} us  {byts/t/1e9:7.0f} GB/s ({byts/t/1e9/peaks['hbm_gbs']:.2f})  {fl/t/1e12:7.0f} TF/s ({fl/t/1e12/peaks['bf16_tflops']:.2f})", flush=True)
for Nt in (16, 64):
    bn = next(b for b in (16,32,64,128,256) if b >= Nt)
    bench(37888, Nt, 3584, 1, 2, bn)
    bench(3584, Nt, 18944, 5, 1, bn)
    bench(4608, Nt, 3584, 4, 1, bn)
for Nt in (128, 256):
    for pair in (1, 2):
        bench(37888, Nt, 3584, 1, 2, Nt, pair=pair)
        bench(3584, Nt, 18944, 5 if pair == 1 else 2, 1, Nt, pair=pair)
        bench(4608, Nt, 3584, 4 if pair == 1 else 2, 1, Nt, pair=pair)
for Nt in (512, 2048, 8192):
    for pair in (1, 2):
        bench(37888, Nt, 3584, 1, 2, 256, iters=10, pair=pair)
        bench(3584, Nt, 18944, 1, 0, 256, iters=10, pair=pair)
for pair in (1, 2):
    bench(8192, 8192, 8192, 1, 0, 256, iters=10, pair=pair)
