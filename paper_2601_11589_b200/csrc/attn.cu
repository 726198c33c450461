// Paged varlen prefill attention — see attn.cuh.
// Math path: bf16 m16n8k16 warp MMAs with ldmatrix from 128-byte-swizzled
// shared memory (the TMA swizzle), online softmax in fp32 (exp2 with the scale
// folded in), quad-shuffle row reductions. KV pages arrive by TMA
// (cp.async.bulk.tensor.3d) into a 2-deep mbarrier ring; the Q tile (a gather
// of (token, head) rows) is loaded once with cp.async.
#include <cstdint>
#include <stdexcept>

#include "attn.cuh"
#include "attn_merge.cuh"
#include "gemm_sm100.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace lp {

namespace {

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// 64 rows of D bf16, stored as D/64 "halves" of [64 rows][128 B] with the TMA
// 128-byte swizzle: 16-byte chunk c of a row sits at (c ^ (row & 7)).
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (chunk >> 3) * (64 * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}


template <int D>
__global__ void __launch_bounds__(128)
    attn_prefill_kernel(const __grid_constant__ CUtensorMap kvm, const AttnCtx c) {
  KTL_SCOPE(kKtlAttnWarp, D);
  constexpr int kChunks = D / 8;           // 16-byte chunks per row
  constexpr int kTileBytes = 64 * D * 2;   // one page of one head
  constexpr int kHalves = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTileBytes;          // [2][tile]
  uint8_t* sV = sK + 2 * kTileBytes;        // [2][tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kTileBytes);

  pdl_trigger();
  const int wi = blockIdx.x;
  const bool live = wi < *c.n_work;  // written by the pre-graph H2D copy
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  if (!live) return;
  const int g = blockIdx.y;
  const int G = c.nq / c.nkv;
  const int4 wk = c.work[wi];
  const int r = wk.x & 0xFFFF, row0 = wk.y;  // high bits: combine entry of a split item
  const int L = c.q_len[r], H = c.hist[r], qs = c.q_start[r];
  const int rows_total = L * G;
  const int* pages = c.page_list + c.page_off[r];
  const size_t ld_q = static_cast<size_t>(c.nq) * D;

  const int row_hi = min(row0 + 63, rows_total - 1);
  const int p_hi = H + row_hi / G;                  // max query position in CTA
  const int p_lo = H + row0 / G;
  const bool partial = wk.w >= 0;
  const int t_begin = wk.z;
  const int t_end = partial ? wk.w : (p_hi + 1 + 63) / 64;

  auto issue_tile = [&](int kt, int buf) {
    const int plane_k = c.kv_plane0 + pages[kt] * 2 * c.nkv + g;
    mbar_arrive_expect_tx(&bars[buf], 2 * kTileBytes);
#pragma unroll
    for (int hf = 0; hf < kHalves; ++hf) {
      tma_load_3d(sK + buf * kTileBytes + hf * 64 * 128, &kvm, &bars[buf], hf * 64, 0, plane_k);
      tma_load_3d(sV + buf * kTileBytes + hf * 64 * 128, &kvm, &bars[buf], hf * 64, 0, plane_k + c.nkv);
    }
  };
  if (tid == 0 && t_begin < t_end) issue_tile(t_begin, 0);

  // ---- Q tile -> smem (rows beyond the member replicate its last row) ----
  const uint32_t sQa = smem_u32(sQ);
  for (int idx = tid; idx < 64 * kChunks; idx += 128) {
    const int rr = idx / kChunks, ch = idx % kChunks;
    const int row = min(row0 + rr, rows_total - 1);
    const int j = row / G, hq = g * G + row % G;
    cp_async16(swz(sQa, rr, ch), c.q + (qs + j) * ld_q + hq * D + ch * 8);
  }
  cp_commit();

  // Per-thread rows: lane/4 and lane/4 + 8 of this warp's 16.
  const int my_row[2] = {row0 + warp * 16 + lane / 4, row0 + warp * 16 + lane / 4 + 8};
  int my_pos[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) my_pos[i] = H + min(my_row[i], rows_total - 1) / G;

  cp_wait_all();
  __syncthreads();
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int rr = warp * 16 + (lane % 16);
    const int ch = ks * 2 + lane / 16;
    ldsm_x4(swz(sQa, rr, ch), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  for (int kt = t_begin; kt < t_end; ++kt) {
    const int it = kt - t_begin, buf = it & 1;
    if (tid == 0 && kt + 1 < t_end) issue_tile(kt + 1, buf ^ 1);  // buf^1 was released by the last barrier
    mbar_wait(&bars[buf], (it >> 1) & 1);
    const uint32_t kb = smem_u32(sK + buf * kTileBytes);
    const uint32_t vb = smem_u32(sV + buf * kTileBytes);

    // S = Q K^T : 16 x 64 per warp.
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-key n-tiles
        const int mi = lane / 8;
        const int key = np * 16 + (mi / 2) * 8 + (lane % 8);
        const int ch = ks * 2 + (mi % 2);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(swz(kb, key, ch), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[ks], b0, b1);
        mma16816(s[2 * np + 1], qf[ks], b2, b3);
      }
    }
    // Causal mask (only tiles crossing the CTA's lowest query position).
    const int kbase = kt * 64;
    if (kbase + 63 > p_lo) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kbase + nt * 8 + (lane % 4) * 2 + (e & 1);
          if (key > my_pos[e >> 1]) s[nt][e] = -INFINITY;
        }
      }
    }
    // Online softmax (rows: e>>1 selects lane/4 or lane/4+8). A split may
    // hold no visible key for some rows: keep them at m = -inf, l = 0.
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * hr], s[nt][2 * hr + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run[hr], mx * c.scale_log2);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      corr[hr] = exp2f(m_run[hr] - m_use);
      m_run[hr] = m_new;
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = ex2_ftz(s[nt][2 * hr] * c.scale_log2 - m_use);
        const float p1 = ex2_ftz(s[nt][2 * hr + 1] * c.scale_log2 - m_use);
        s[nt][2 * hr] = p0;
        s[nt][2 * hr + 1] = p1;
        sum += p0 + p1;
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      l_run[hr] = l_run[hr] * corr[hr] + sum;
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // 16 keys per k-step
      uint32_t a[4];
      a[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
      a[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
      a[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      a[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {  // pairs of 8-dim n-tiles
        const int mi = lane / 8;
        const int key = ks * 16 + (mi % 2) * 8 + (lane % 8);
        const int ch = dp * 2 + (mi / 2);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(swz(vb, key, ch), b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();  // every warp is done with `buf` before it is refilled
  }

  if (!partial) {
    // Normalise and store valid rows.
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int row = my_row[hr];
      if (row >= rows_total) continue;
      const int j = row / G, hq = g * G + row % G;
      const float inv = 1.f / l_run[hr];
      __nv_bfloat16* dst = c.out + (qs + j) * ld_q + hq * D;
#pragma unroll
      for (int nt = 0; nt < D / 8; ++nt) {
        const int col = nt * 8 + (lane % 4) * 2;
        *reinterpret_cast<uint32_t*>(dst + col) = pack_bf16(o[nt][2 * hr] * inv, o[nt][2 * hr + 1] * inv);
      }
    }
  } else {
    // Unnormalised partial + (m, l) for the combine kernel.
    const size_t slab = static_cast<size_t>(wi) * c.nkv + g;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rl = warp * 16 + lane / 4 + hr * 8;
      float* dst = c.ws_o + (slab * 64 + rl) * D;
#pragma unroll
      for (int nt = 0; nt < D / 8; ++nt) {
        const int col = nt * 8 + (lane % 4) * 2;
        *reinterpret_cast<float2*>(dst + col) = make_float2(o[nt][2 * hr], o[nt][2 * hr + 1]);
      }
      if ((lane & 3) == 0) {
        c.ws_ml[(slab * 64 + rl) * 2 + 0] = m_run[hr];
        c.ws_ml[(slab * 64 + rl) * 2 + 1] = l_run[hr];
      }
    }
  }
}


// Merge grid: (row blocks that were split, nkv, block_rows / 8), one warp per row.
template <int D>
__global__ void __launch_bounds__(256) attn_combine_kernel(const AttnCtx c) {
  KTL_SCOPE(kKtlAttnCombine, 0);
  pdl_trigger();
  const int ci = blockIdx.x;
  const bool live = ci < *c.n_combine;
  pdl_wait();
  if (!live) return;
  const int4 e = c.combine[ci];
  merge_row<D>(c, e.z, e.w, blockIdx.y, e.x, e.y, blockIdx.z * 8 + threadIdx.x / 32, threadIdx.x % 32);
}

template <int D>
void launch(const AttnCtx& c, const CUtensorMap& kvm, int work_cap, int combine_cap, bool with_combine,
            cudaStream_t st) {
  constexpr int smem = 1024 + 5 * 64 * D * 2 + 64;
  smem_attr_once(reinterpret_cast<const void*>(attn_prefill_kernel<D>), smem);
  launch_k(attn_prefill_kernel<D>, dim3(work_cap, c.nkv), dim3(128), smem, st, kvm, c);
  // Graph-bucket shapes split long histories into many short key ranges
  // (up to 32 per 64-row block): a separate merge grid (one warp per row,
  // many CTAs) beats a serial merge by the last split CTA.
  if (with_combine) launch_k(attn_combine_kernel<D>, dim3(combine_cap, c.nkv, c.block_rows / 8), dim3(256), 0, st, c);
}

}  // namespace

CUtensorMap make_kv_tmap(const void* pool, int64_t planes, int head_dim) {
  const uint64_t dims[3] = {static_cast<uint64_t>(head_dim), 64, static_cast<uint64_t>(planes)};
  const uint64_t strides[2] = {static_cast<uint64_t>(head_dim) * 2, static_cast<uint64_t>(64) * head_dim * 2};
  const uint32_t box[3] = {64, 64, 1};
  return make_tmap_3d_bf16(pool, dims, strides, box);
}

void attention_prefill(const AttnCtx& c, const CUtensorMap& kv_map, int head_dim, int work_cap,
                       int combine_cap, cudaStream_t st, bool with_combine) {
  if (debug_empty("attn")) return launch_empty(dim3(work_cap), dim3(128), st);
  if (head_dim == 128 && c.block_rows == kAttnTcRows) {
    attention_prefill_tc(c, kv_map, work_cap, st);
  } else if (head_dim == 128) {
    launch<128>(c, kv_map, work_cap, combine_cap, with_combine, st);
  } else if (head_dim == 64) {
    launch<64>(c, kv_map, work_cap, combine_cap, with_combine, st);
  } else {
    throw std::runtime_error("attention: head_dim must be 64 or 128");
  }
}

}  // namespace lp

KTL_EXPORT(attn)
