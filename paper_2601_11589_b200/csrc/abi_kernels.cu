// Kernel-level C-ABI test hooks (declared in include/laps_prefill_testing.h). These let
// the parity tests drive each sm_100a kernel on raw device pointers without
// going through a full instance. Product callers use include/laps_prefill.h.
#include <cstdio>
#include <stdexcept>
#include <string>

#include "abi_common.h"
#include "gemm_sm100.cuh"

using namespace lp;

extern "C" {

int lpk_gemm(const void* W, const void* X, void* out, float* ws, const void* bias, int M, int N,
             int K, int splits, int mode, int bn, int ldo, const int* n_dev, void* stream, int pair) {
  return lp_guard([&] {
    const CUtensorMap ta = make_tmap_bf16(W, M, K, 128);
    const CUtensorMap tb = make_tmap_bf16(X, N, K, gemm_b_box_rows(bn, pair));
    GemmArgs a;
    a.M = M;
    a.N = N;
    a.K = K;
    a.splits = splits;
    a.n_dev = n_dev;
    a.mode = mode;
    a.out = out;
    a.ldo = ldo;
    a.bias = bias;
    a.ws = ws;
    a.ws_stride = N;
    gemm_launch(ta, tb, a, bn, static_cast<cudaStream_t>(stream), 0, pair);
    lp_check(cudaGetLastError(), "gemm launch");
  });
}

int lpk_gemm_stream_k(const void* W, const void* X, float* ws, int M, int N, int K, int bn, int pair,
                      const int* n_dev, int* seg_table, int max_ctas, void* stream) {
  return lp_guard([&] {
    const CUtensorMap ta = make_tmap_bf16(W, M, K, 128);
    const CUtensorMap tb = make_tmap_bf16(X, N, K, gemm_b_box_rows(bn, pair));
    GemmArgs a;
    a.M = M;
    a.N = N;
    a.K = K;
    a.splits = -1;
    a.n_dev = n_dev;
    a.mode = kEpiF32Partial;
    a.ws = ws;
    a.ws_stride = N;
    a.sk_tab = seg_table;
    gemm_launch(ta, tb, a, bn, static_cast<cudaStream_t>(stream), max_ctas, pair);
    lp_check(cudaGetLastError(), "gemm launch");
  });
}

}  // extern "C"
