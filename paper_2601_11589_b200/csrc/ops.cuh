// Fused elementwise / row kernels around the tcgen05 GEMMs (north_star
// subsystem 3): embedding + RMSNorm, split-K reduction + bias + RoPE + paged
// KV append, split-K reduction + residual + RMSNorm, last-token gather, argmax,
// and deterministic weight initialisation.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lp {

using bf16 = __nv_bfloat16;

// Weight init: dst[i] = bf16(synth_weight_f32(seed, tensor_id, logical(i), scale)).
// interleave_rows > 0: dst is the [2*rows, cols] gate/up interleave of two
// logical tensors (tensor_id = gate, tensor_id+1 = up), each [rows, cols].
void init_weights(bf16* dst, size_t n, uint64_t seed, uint64_t tensor_id, float scale,
                  int interleave_rows, int cols, cudaStream_t st);
void fill_bf16(bf16* dst, size_t n, float v, cudaStream_t st);

// Session-KV migration: copy `n_pages` pages of every layer from one paged
// pool to another (page ids in device memory). `src_pool` may be a peer
// device's pool (read over NVLink with peer access enabled). One launch moves
// the whole session: grid (pages, layers), 16-byte vector copies.
void kv_page_copy(const bf16* src_pool, size_t src_layer_stride, bf16* dst_pool, size_t dst_layer_stride,
                  size_t page_elems, const int* src_pages, const int* dst_pages, int n_pages, int layers,
                  cudaStream_t st);

struct RowCtx {
  const int* n_live;  // device scalar: live tokens
  int t_cap;          // grid size (tokens) the launch was built for
  int h;
  float eps;
};

// x_resid[t] = embed[tok[t]] (fp32); x_norm[t] = bf16(rmsnorm(x_resid[t]) * gamma)
void embed_rmsnorm(const RowCtx& c, const int* tokens, const bf16* embed, const bf16* gamma,
                   float* x_resid, bf16* x_norm, cudaStream_t st);

// x_resid[t] += sum_s ws[s][t]; x_norm[t] = bf16(rmsnorm(x_resid[t]) * gamma)
// splits_dev (optional): device-side split count overriding `splits`.
void resid_rmsnorm(const RowCtx& c, const float* ws, int splits, const int* splits_dev, const int* sk_tab,
                   size_t ws_stride_rows,
                   float* x_resid, const bf16* gamma, bf16* x_norm, cudaStream_t st);

struct QkvCtx {
  const int* n_live;
  int t_cap;
  int nq, nkv, d;
  int page_size;
  const float* ws;           // [splits][t_cap][qkv_out] fp32 partials
  int splits;
  const int* splits_dev;     // optional device-side split count (overrides `splits`)
  size_t ws_stride_rows;
  const bf16* bias;          // [qkv_out]
  const int* positions;      // [T] absolute position
  const int* slot_mapping;   // [T] page * page_size + slot
  const float* inv_freq;     // [d/2]
  bf16* q_out;               // [T, nq*d]
  bf16* kv_layer;            // layer base of the paged cache
  int s_cap = 8;             // upper bound of the split count (picks the load schedule)
  const int* sk_tab = nullptr;  // stream-K segment table (*splits_dev < 0; gemm_sm100.cuh kSkTab*)
};
// reduce splits + bias; RoPE(q, k); q -> q_out; k, v -> paged cache
void qkv_post(const QkvCtx& c, cudaStream_t st);

// x_last[r] = x_norm[last_idx[r]]; also zeroes argmax_keys[r].
void gather_rows(const int* n_rows, int r_cap, const int* idx, const bf16* src, bf16* dst, int h,
                 unsigned long long* argmax_keys, cudaStream_t st);
// keys[r] = max over j of an order-preserving (logit, -j) key: the greedy
// first token is 0x7fffffff - (key & 0xffffffff) (lowest index on ties).
void argmax_rows(const int* n_rows, int r_cap, const float* logits, int vocab, unsigned long long* keys,
                 cudaStream_t st);
inline int32_t argmax_token(unsigned long long key) {
  return static_cast<int32_t>(0x7fffffffu - static_cast<uint32_t>(key & 0xffffffffull));
}

}  // namespace lp
