// Varlen paged causal prefill attention with GQA (north_star subsystem 1).
//
// Each request r contributes L_r new query tokens at positions
// [H_r, H_r + L_r); token j attends to cached + new keys at positions
// 0 .. H_r + j (the alpha*L*(L+2H) and gamma_r*H terms of the reference cost
// model, cost_model.cpp:36-41). Keys/values live in the paged cache, one
// 64-token page == one key tile, so a CTA streams its request's page list.
//
// Work decomposition: rows = (token, q-head) pairs of one KV head's query
// group packed together ("GQA packing"), 64 rows per CTA, so every K/V page a
// CTA loads is reused by all G query heads that share it. The grid is built
// from capacity (T_cap, R_cap), never from H, so the launch can sit inside a
// CUDA graph; live work items come from device memory.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lp {

struct AttnCtx {
  const int* n_work;      // device scalar: live work items
  const int2* work;       // [W]: (member r, first packed row of this CTA)
  const int* q_start;     // [R]: packed index of member's first new token
  const int* q_len;       // [R]: L_r
  const int* hist;        // [R]: H_r
  const int* page_list;   // flattened page ids of every member
  const int* page_off;    // [R]: member r's pages start at page_list[page_off[r]]
  const __nv_bfloat16* q;        // [T, nq*d]
  const __nv_bfloat16* kv_layer; // this layer's paged cache
  __nv_bfloat16* out;            // [T, nq*d]
  int nq, nkv;
  float scale_log2;  // log2(e) / sqrt(d)
};

constexpr int kAttnRows = 64;   // rows per CTA
constexpr int kAttnPage = 64;   // required page size (== key tile)

// grid_x = work capacity, grid_y = nkv. head_dim in {64, 128}.
void attention_prefill(const AttnCtx& c, int head_dim, int work_cap, cudaStream_t st);

}  // namespace lp
