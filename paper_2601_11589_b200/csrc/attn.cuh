// Varlen paged causal prefill attention with GQA (north_star subsystem 1).
//
// Each request r contributes L_r new query tokens at positions
// [H_r, H_r + L_r); token j attends to cached + new keys at positions
// 0 .. H_r + j (the alpha*L*(L+2H) and gamma_r*H terms of the reference cost
// model, cost_model.cpp:36-41). Keys/values live in the paged cache, one
// 64-token page == one key tile, staged into shared memory by TMA (one 3-D
// tensor map over the whole pool, 128-byte swizzle) behind an mbarrier
// double buffer.
//
// Work decomposition: rows = (token, q-head) pairs of one KV head's query
// group ("GQA packing", 64 rows per CTA) so every page a CTA loads is reused
// by all G query heads that share it. A work item is (member, row block, key
// tile range): short batches over long histories are split along the key
// range (flash-decoding style) and merged afterwards — by a merge grid on
// the graph path (attn.cu; graph variants without it replay batches that did
// not split), by the last split CTA of the block in the tcgen05 kernel — so
// the grid fills the GPU even when few rows exist. Items are ordered heaviest
// first.
// The grid is sized from capacity, never from H, so it lives inside the
// per-shape CUDA graphs; the live work list comes from device memory.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lp {

struct AttnCtx {
  const int* n_work;      // device scalar: live work items
  const int4* work;       // [W]: (member r, first packed row, tile begin, tile end or -1 = causal end)
  const int* n_combine;   // device scalar: row blocks that were split
  const int4* combine;    // [C]: (member r, first packed row, first work item, n splits)
  const int* q_start;     // [R]: packed index of member's first new token
  const int* q_len;       // [R]: L_r
  const int* hist;        // [R]: H_r
  const int* page_list;   // flattened page ids of every member
  const int* page_off;    // [R]: member r's pages start at page_list[page_off[r]]
  const __nv_bfloat16* q;        // [T, nq*d]
  int kv_plane0;                 // first TMA plane of this layer (layer * n_pages * 2 * nkv)
  __nv_bfloat16* out;            // [T, nq*d]
  float* ws_o;                   // split partials [W][nkv][64][d] fp32 (unnormalised)
  float* ws_ml;                  // [W][nkv][64][2] running max (log2 units) and sum
  int nq, nkv;
  float scale_log2;  // log2(e) / sqrt(d)
  int block_rows;    // rows per work item: 64 (warp-MMA kernel) or 128 (tcgen05 kernel)
  int* comb_cnt = nullptr;  // [combine capacity][nkv] split arrival tickets (zero between launches)
  // Persistent tcgen05 schedule (attn_tc.cu): work[i] = (member, first row,
  // first page, end page) of piece i, work2[i] = (kv head, combine entry or -1,
  // partial slot, 0); CTA b runs pieces [cta_off[b], cta_off[b + 1]).
  const int4* work2 = nullptr;
  const int* cta_off = nullptr;
};

constexpr int kAttnRows = 64;    // rows per CTA
constexpr int kAttnPage = 64;    // required page size (== key tile)
constexpr int kAttnSplitCap = 1024;  // max split (partial) work items per forward
constexpr int kAttnTcRows = 128;     // rows per CTA of the tcgen05 kernel (head_dim 128)
constexpr int kAttnMaxCtas = 256;    // persistent tcgen05 grid: one CTA per SM

// TMA map over the whole paged pool viewed as [planes][64 slots][d] bf16,
// plane = (layer * n_pages + page) * 2 * nkv + (is_v * nkv + kv_head).
CUtensorMap make_kv_tmap(const void* pool, int64_t planes, int head_dim);

// grid_x = work capacity, grid_y = nkv. head_dim in {64, 128}. with_combine = false
// drops the graph path's merge grid (a launch with no key-range splits).
void attention_prefill(const AttnCtx& c, const CUtensorMap& kv_map, int head_dim, int work_cap,
                       int combine_cap, cudaStream_t st, bool with_combine = true);
// tcgen05/TMEM kernel (head_dim 128, block_rows 128); see attn_tc.cu.
void attention_prefill_tc(const AttnCtx& c, const CUtensorMap& kv_map, int work_cap, cudaStream_t st);
// Persistent variant: n_cta CTAs walk the balanced piece lists of the
// schedule (work / work2 / cta_off), partial pieces merged by the last one.
void attention_prefill_tc_persistent(const AttnCtx& c, const CUtensorMap& kv_map, int n_cta, cudaStream_t st);

}  // namespace lp
