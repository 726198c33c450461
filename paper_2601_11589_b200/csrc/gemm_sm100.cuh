// tcgen05/TMEM bf16 GEMM for the prefill projections (QKV, O, gate/up, down,
// LM head). Swap-AB orientation: the WEIGHT matrix W[M=out_features, K] is the
// MMA "A" operand (M = 128 rows per tile) and the token activations X[T, K]
// are the "B" operand (N = tokens per tile, 16..256). So
//     D[m, n] = sum_k W[m, k] * X[n, k]        (Y^T = W X^T)
// Both operands are K-major, staged by TMA with 128-byte swizzle; the fp32
// accumulator lives in TMEM (double-buffered so the epilogue of tile i
// overlaps the mainloop of tile i+1). Persistent grid: one CTA per SM walks
// (split, m_tile, n_tile) work units.
//
// For the short-prefill regime (T <= 256 tokens) the kernel is a weight
// streamer: HBM-bound at T*... flop/byte well under the ridge; split-K keeps
// all 148 SMs pulling weights when M/128 is small (O, down, QKV projections).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace lp {

enum GemmEpilogue : int {
  kEpiBf16 = 0,        // out_bf16[n*ldo + m] = acc (+ bias[m])
  kEpiF32Partial = 1,  // ws[(split*ws_stride + n)*M + m] = acc
  kEpiSiluMul = 2,     // rows interleaved (gate,up): out_bf16[n*ldo + m/2] = silu(g)*u
  kEpiF32 = 3,         // out_f32[n*ldo + m] = acc
  kEpiQkvRope = 4,     // q/k/v = bf16(RoPE(acc + bias)): q -> q_out, k/v -> paged KV slot (split-K = 1)
  kEpiResidAdd = 5,    // resid_f32[n*M + m] += acc (split-K = 1)
};

// Extra operands of the fused QKV epilogue (kEpiQkvRope). head_dim == 128:
// one 128-row weight tile is exactly one head.
struct QkvEpi {
  const int* positions = nullptr;  // [T] absolute positions
  const int* slots = nullptr;      // [T] page * page_size + slot
  const float* inv_freq = nullptr; // [64]
  void* q_out = nullptr;           // bf16 [T, nq*128]
  void* kv_layer = nullptr;        // bf16 paged cache of this layer
  int nq = 0, nkv = 0, page_size = 64;
};

// Stream-K segment table, written by the GEMM, read by the reduction kernels:
// [0] token-tile width, [1] token tiles, [2] weight rows per tile, [3] unused,
// [kSkTabHeader + m_tile * tiles + n_tile] segments of that output tile.
constexpr int kSkTabHeader = 4;

struct GemmArgs {
  int M = 0;            // weight rows (output features)
  int N = 0;            // token capacity (rows of X)
  int K = 0;            // reduction length (multiple of 64)
  int splits = 1;       // split-K factor
  // Optional device-side split-K factor (overrides `splits`). A value < 0
  // selects stream-K (kEpiF32Partial only): every CTA (pair) takes an equal
  // share of the flattened (tile, K-block) space, so a tile is cut into 1..n
  // segments at share boundaries; segment j lands in ws slice j and the
  // tile's segment count in sk_tab, and the reduction kernel (qkv_post /
  // resid_rmsnorm) sums slices 0..nseg-1 of each element in order.
  const int* splits_dev = nullptr;
  int* sk_tab = nullptr;  // stream-K segment table (layout: kSkTab*)
  const int* n_dev = nullptr;  // optional device-side live token count (<= N)
  // Optional device-side token-tile count (per-batch tile plan; clamped to
  // [ceil(n_live / bn), ceil(n_live / 16)]); n_tiles_cap bounds it for the grid.
  const int* ntiles_dev = nullptr;
  int n_tiles_cap = 0;
  int mode = kEpiBf16;
  void* out = nullptr;
  int ldo = 0;
  const void* bias = nullptr;  // bf16[M] (kEpiBf16 only)
  float* ws = nullptr;
  int ws_stride = 0;    // rows per split slice in ws (>= N)
  float* resid = nullptr;  // kEpiResidAdd target [N, M] fp32
  QkvEpi qkv;              // kEpiQkvRope operands
};

// Build a 2D bf16 tensor map over a row-major [rows, cols] matrix, box
// [box_rows, 64 cols], 128-byte swizzle.
CUtensorMap make_tmap_bf16(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
// 3-D bf16 tensor map, 128-byte swizzle (dims innermost first).
CUtensorMap make_tmap_3d_bf16(const void* ptr, const uint64_t dims[3], const uint64_t strides_bytes[2],
                              const uint32_t box[3]);

// Launch. `bn` is the token-tile width (16, 32, 64, 128 or 256). pair = 2
// selects the CTA-pair (cta_group::2, M = 256 per pair) variant; M must then
// be a multiple of 256 and bn >= 32. tmB must have been built with
// box_rows == gemm_b_box_rows(bn, pair) (= bn / pair).
void gemm_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, int bn,
                 cudaStream_t stream, int max_ctas = 0, int pair = 1);
int gemm_b_box_rows(int bn, int pair);

int num_sms();

}  // namespace lp
