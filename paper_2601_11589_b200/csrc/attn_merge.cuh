// Split-KV merge: merge_row is shared by the graph-path combine grid
// (attn.cu) and the tcgen05 kernel, whose last split CTA of a row block merges
// the block itself (few, long splits: no separate combine launch between
// attention and the O projection).
#pragma once
#include <cuda_bf16.h>

#include "attn.cuh"

namespace lp {

// Merge the key-range splits of one row of a split (row block, kv head):
// lane s fetches split s's (m, l) (<= 32 splits), weights come from warp
// reductions, and the partial O rows are read 8 splits at a time with all
// loads in flight.
template <int D>
__device__ __forceinline__ void merge_row(const AttnCtx& c, int first, int ns, int g, int r, int row0, int rl,
                                          int lane) {
  const int G = c.nq / c.nkv;
  const int rows_total = c.q_len[r] * G, qs = c.q_start[r];
  const int br = c.block_rows;
  const int row = row0 + rl;
  if (rl >= br || row >= rows_total) return;
  float m = -INFINITY, l = 0.f;
  if (lane < ns) {
    const size_t slab = static_cast<size_t>(first + lane) * c.nkv + g;
    m = __ldcg(c.ws_ml + (slab * br + rl) * 2);
    l = __ldcg(c.ws_ml + (slab * br + rl) * 2 + 1);
  }
  float m_star = m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m_star = fmaxf(m_star, __shfl_xor_sync(0xffffffffu, m_star, o));
  const float w_mine = (lane < ns && m != -INFINITY) ? exp2f(m - m_star) : 0.f;
  float lsum = w_mine * l;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  constexpr int kV = D / 32;
  float acc[kV];
#pragma unroll
  for (int k = 0; k < kV; ++k) acc[k] = 0.f;
  const size_t split_stride = static_cast<size_t>(c.nkv) * br * D;
  const float* base = c.ws_o + ((static_cast<size_t>(first) * c.nkv + g) * br + rl) * D + lane;
  for (int s0 = 0; s0 < ns; s0 += 8) {
    float x[8][kV];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#pragma unroll
      for (int k = 0; k < kV; ++k) x[q][k] = s0 + q < ns ? __ldcg(base + (s0 + q) * split_stride + k * 32) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float w = __shfl_sync(0xffffffffu, w_mine, (s0 + q) & 31);
#pragma unroll
      for (int k = 0; k < kV; ++k) acc[k] += w * x[q][k];
    }
  }
  const size_t ld_q = static_cast<size_t>(c.nq) * D;
  const int j = row / G, hq = g * G + row % G;
  __nv_bfloat16* dst = c.out + (qs + j) * ld_q + hq * D;
  const float inv = 1.f / lsum;
#pragma unroll
  for (int k = 0; k < kV; ++k) dst[k * 32 + lane] = __float2bfloat16_rn(acc[k] * inv);
}

// Block merge for the last split CTA: every thread takes (row, 16-column)
// items, so all rows of the block are merged in one round of loads (the
// splits' (m, l) and partial O columns of an item are all in flight at once)
// instead of one warp walking the rows one after another.
template <int D>
__device__ __forceinline__ void merge_block(const AttnCtx& c, int first, int ns, int g, int r, int row0) {
  const int G = c.nq / c.nkv;
  const int rows_total = c.q_len[r] * G, qs = c.q_start[r];
  const int br = c.block_rows;
  constexpr int kC = 16, kQ = D / kC, kS = 4;
  const size_t split_o = static_cast<size_t>(c.nkv) * br * D;
  const size_t split_ml = static_cast<size_t>(c.nkv) * br * 2;
  const size_t ld_q = static_cast<size_t>(c.nq) * D;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = threadIdx.x; it < br * kQ; it += blockDim.x) {
    const int rl = it / kQ, q = it % kQ;
    const int row = row0 + rl;
    if (row >= rows_total) continue;
    const size_t brow = (static_cast<size_t>(first) * c.nkv + g) * br + rl;
    float acc[kC];
#pragma unroll
    for (int i = 0; i < kC; ++i) acc[i] = 0.f;
    float m_acc = -INFINITY, l_acc = 0.f;
    for (int s0 = 0; s0 < ns; s0 += kS) {
      float m[kS], l[kS];
      float4 x[kS][kC / 4];
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const bool on = s0 + s < ns;
        m[s] = on ? __ldcg(c.ws_ml + brow * 2 + (s0 + s) * split_ml) : -INFINITY;
        l[s] = on ? __ldcg(c.ws_ml + brow * 2 + (s0 + s) * split_ml + 1) : 0.f;
        const float4* src = reinterpret_cast<const float4*>(c.ws_o + brow * D + (s0 + s) * split_o + q * kC);
#pragma unroll
        for (int v = 0; v < kC / 4; ++v) x[s][v] = on ? __ldcg(src + v) : zero;
      }
      float ms = m_acc;
#pragma unroll
      for (int s = 0; s < kS; ++s) ms = fmaxf(ms, m[s]);
      const float keep = (m_acc == -INFINITY) ? 0.f : exp2f(m_acc - ms);
      l_acc *= keep;
#pragma unroll
      for (int i = 0; i < kC; ++i) acc[i] *= keep;
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const float w = (m[s] == -INFINITY) ? 0.f : exp2f(m[s] - ms);
        l_acc += w * l[s];
#pragma unroll
        for (int v = 0; v < kC / 4; ++v) {
          acc[4 * v + 0] += w * x[s][v].x;
          acc[4 * v + 1] += w * x[s][v].y;
          acc[4 * v + 2] += w * x[s][v].z;
          acc[4 * v + 3] += w * x[s][v].w;
        }
      }
      m_acc = ms;
    }
    const float inv = 1.f / l_acc;
    const int j = row / G, hq = g * G + row % G;
    uint4 w[2];
    __nv_bfloat162* wp = reinterpret_cast<__nv_bfloat162*>(w);
#pragma unroll
    for (int i = 0; i < kC / 2; ++i) wp[i] = __floats2bfloat162_rn(acc[2 * i] * inv, acc[2 * i + 1] * inv);
    uint4* dst = reinterpret_cast<uint4*>(c.out + (qs + j) * ld_q + hq * D + q * kC);
    dst[0] = w[0];
    dst[1] = w[1];
  }
}

// Called by every thread of a CTA that wrote a split partial (work item wi,
// kv head g) after its partial stores: the last split of the row block to
// arrive (atomic ticket per (combine entry, kv head), reset by that CTA for
// the next launch / graph replay) merges all splits' rows with its warps.
template <int D>
__device__ __forceinline__ void attn_merge_if_last(const AttnCtx& c, int wi, int g, int n_warps, int* scratch) {
  int& s_last = scratch[1];
  __threadfence();
  __syncthreads();
  const int ci = c.work[wi].x >> 16;  // the block's combine entry (packed by the host)
  if (threadIdx.x == 0) {
    const int ns = c.combine[ci].w;
    int* cnt = c.comb_cnt + static_cast<size_t>(ci) * c.nkv + g;
    const int old = atomicAdd(cnt, 1);
    const int last = old == ns - 1;
    if (last) *cnt = 0;
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int4 e = c.combine[ci];
  (void)n_warps;
  merge_block<D>(c, e.z, e.w, g, e.x, e.y);
}


}  // namespace lp
