// Paged varlen prefill attention — see attn.cuh.
// v1 math path: bf16 m16n8k16 warp MMAs with ldmatrix from XOR-swizzled
// shared memory, cp.async double-buffered page loads, online softmax in fp32
// (exp2 with the scale folded in), quad-shuffle row reductions.
#include <cstdint>

#include "attn.cuh"
#include "launch.cuh"

namespace lp {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

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

// Row of D bf16 = D/8 16-byte chunks; chunk c of row r lives at c ^ (r & 7).
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + row * (D * 2) + ((chunk ^ (row & 7)) << 4);
}

template <int D>
__global__ void __launch_bounds__(128)
    attn_prefill_kernel(const AttnCtx c) {
  constexpr int kChunks = D / 8;           // 16-byte chunks per row
  constexpr int kTileBytes = 64 * D * 2;   // one page of one head
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTileBytes;          // [2][64][D]
  uint8_t* sV = sK + 2 * kTileBytes;        // [2][64][D]

  pdl_trigger();
  const int wi = blockIdx.x;
  const bool live = wi < *c.n_work;  // written by the pre-graph H2D copy
  pdl_wait();
  if (!live) return;
  const int g = blockIdx.y;
  const int G = c.nq / c.nkv;
  const int2 wk = c.work[wi];
  const int r = wk.x, row0 = wk.y;
  const int L = c.q_len[r], H = c.hist[r], qs = c.q_start[r];
  const int rows_total = L * G;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int* pages = c.page_list + c.page_off[r];
  const size_t page_elems = static_cast<size_t>(2) * c.nkv * kAttnPage * D;
  const size_t ld_q = static_cast<size_t>(c.nq) * D;

  // ---- Q tile -> smem (rows beyond the member replicate its last row) ----
  const uint32_t sQa = static_cast<uint32_t>(__cvta_generic_to_shared(sQ));
  for (int idx = tid; idx < 64 * kChunks; idx += 128) {
    const int rr = idx / kChunks, ch = idx % kChunks;
    const int row = min(row0 + rr, rows_total - 1);
    const int j = row / G, hq = g * G + row % G;
    const __nv_bfloat16* src = c.q + (qs + j) * ld_q + hq * D + ch * 8;
    cp_async16(sQ + (swz<D>(sQa, rr, ch) - sQa), src);
  }
  cp_commit();

  const int row_hi = min(row0 + 63, rows_total - 1);
  const int p_hi = H + row_hi / G;                  // max query position in CTA
  const int n_tiles = (p_hi + 1 + 63) / 64;
  const int p_lo = H + row0 / G;

  auto load_kv = [&](int kt, int buf) {
    const size_t pbase = static_cast<size_t>(pages[kt]) * page_elems;
    const __nv_bfloat16* kp = c.kv_layer + pbase + static_cast<size_t>(g) * kAttnPage * D;
    const __nv_bfloat16* vp = c.kv_layer + pbase + static_cast<size_t>(c.nkv + g) * kAttnPage * D;
    const uint32_t kb = static_cast<uint32_t>(__cvta_generic_to_shared(sK + buf * kTileBytes));
    const uint32_t vb = static_cast<uint32_t>(__cvta_generic_to_shared(sV + buf * kTileBytes));
    for (int idx = tid; idx < 64 * kChunks; idx += 128) {
      const int rr = idx / kChunks, ch = idx % kChunks;
      cp_async16(sK + buf * kTileBytes + (swz<D>(kb, rr, ch) - kb), kp + rr * D + ch * 8);
      cp_async16(sV + buf * kTileBytes + (swz<D>(vb, rr, ch) - vb), vp + rr * D + ch * 8);
    }
    cp_commit();
  };
  load_kv(0, 0);

  // Per-thread rows: lane/4 and lane/4 + 8 of this warp's 16.
  const int my_row[2] = {row0 + warp * 16 + lane / 4, row0 + warp * 16 + lane / 4 + 8};
  int my_pos[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) my_pos[i] = H + min(my_row[i], rows_total - 1) / G;

  cp_wait<1>();  // Q landed
  __syncthreads();
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int rr = warp * 16 + (lane % 16);
    const int ch = ks * 2 + lane / 16;
    ldsm_x4(swz<D>(sQa, rr, ch), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  for (int kt = 0; kt < n_tiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_tiles) {
      load_kv(kt + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t kb = static_cast<uint32_t>(__cvta_generic_to_shared(sK + buf * kTileBytes));
    const uint32_t vb = static_cast<uint32_t>(__cvta_generic_to_shared(sV + buf * kTileBytes));

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
        ldsm_x4(swz<D>(kb, key, ch), b0, b1, b2, b3);
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
    // Online softmax (rows: e>>1 selects lane/4 or lane/4+8).
    float corr[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * hr], s[nt][2 * hr + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run[hr], mx * c.scale_log2);
      corr[hr] = exp2f(m_run[hr] - m_new);
      m_run[hr] = m_new;
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = exp2f(s[nt][2 * hr] * c.scale_log2 - m_new);
        const float p1 = exp2f(s[nt][2 * hr + 1] * c.scale_log2 - m_new);
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
        ldsm_x4_t(swz<D>(vb, key, ch), b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();  // buffer `buf` is refilled next iteration
  }

  // Normalise and store valid rows.
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int row = my_row[hr];
    if (row >= rows_total || row > row0 + 63) continue;
    const int j = row / G, hq = g * G + row % G;
    const float inv = 1.f / l_run[hr];
    __nv_bfloat16* dst = c.out + (qs + j) * ld_q + hq * D;
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt) {
      const int col = nt * 8 + (lane % 4) * 2;
      *reinterpret_cast<uint32_t*>(dst + col) =
          pack_bf16(o[nt][2 * hr] * inv, o[nt][2 * hr + 1] * inv);
    }
  }
}

}  // namespace

void attention_prefill(const AttnCtx& c, int head_dim, int work_cap, cudaStream_t st) {
  const dim3 grid(work_cap, c.nkv);
  if (head_dim == 128) {
    constexpr int smem = 5 * 64 * 128 * 2;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(attn_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      set = true;
    }
    launch_k(attn_prefill_kernel<128>, grid, dim3(128), smem, st, c);
  } else {
    constexpr int smem = 5 * 64 * 64 * 2;
    launch_k(attn_prefill_kernel<64>, grid, dim3(128), smem, st, c);
  }
}

}  // namespace lp
