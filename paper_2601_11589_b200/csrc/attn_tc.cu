// tcgen05/TMEM prefill attention (head_dim 128) — the dense path for long
// prompts and deep batches (north_star subsystem 2: "tcgen05/TMEM bf16 GEMMs
// ... and for long-prompt attention").
//
// One CTA = 128 packed (token, q-head) rows of one KV group x a key range.
// Roles (320 threads = 10 warps, kThreads):
//   warp 0   TMA producers (lane 0 K, lane 1 V): pages (2 pages = 128 keys
//            per step) into separate 3-stage K and V rings, laid out
//            [d-half][128 keys][128 B] (128B swizzle);
//   warp 1   MMA issuer (one thread):  S = Q K^T into TMEM (double-buffered,
//            so S(j+1) overlaps the softmax of j), then O += P V with V as an
//            MN-major operand (no transpose pass) and O resident in TMEM;
//   warps 2-9 softmax, two warpgroups: query row = TMEM lane (warp % 4
//            selects the lane quarter), group 0 owns key/d columns 0-63 and
//            group 1 columns 64-127 of that row, so each thread does half a
//            row per step. tcgen05.ld of its S half, causal mask, row max
//            exchanged with the partner thread through smem (one named
//            barrier per quarter per step), online softmax in the log2 domain
//            with LAZY rescaling (the reference max moves only when a row max
//            grows by > 2^8, so O in TMEM is rarely touched), P -> TMEM (bf16
//            pairs; the PV MMA reads its A operand from tensor memory, so no
//            smem round trip or async-proxy fence sits in the step);
//            epilogue O / l -> bf16 (or fp32 partial for key splits).
// TMEM (512 columns): S[2] 0 / 128, O 256, P[2] 384 / 448 (64 packed columns
// each; double-buffered, so softmax of step j+1 waits only for the PV two
// steps back that read the same buffer).
// Numerics match the mma.sync path (and the oracle's storage points): fp32
// scores, bf16 P, fp32 O accumulation; key tiles of 128 instead of 64 change
// only the online-softmax rescale points.
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <stdexcept>

#include "attn.cuh"
#include "attn_merge.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace lp {

namespace {

constexpr int kD = 128;
constexpr int kRows = 128;
constexpr int kKeys = 128;                 // keys per step (2 pages)
constexpr int kHalfBytes = kRows * 128;    // [128 rows][64 elems] bf16 = 16 KiB
constexpr int kQBytes = 2 * kHalfBytes;    // Q / P / K / V tile: 32 KiB each
constexpr int kKStages = 3;  // K runs a step further ahead (S(s+2) is issued right after PV(s))
constexpr int kVStages = 3;
constexpr int kThreads = 320;
constexpr int kSoftmaxWarps = 8;
constexpr float kRescaleTau = 8.0f;  // log2 units: P <= 2^8 between rescales

struct TcSmem {
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;                 // [stage][32 KiB]
  static constexpr int kV = kK + kKStages * kQBytes;      // [stage][32 KiB]
  static constexpr int kBars = kV + kVStages * kQBytes;
  static constexpr int kRed = kBars + 256;                // float [2 parity][2 group][128 rows]
  static constexpr int kTotal = kRed + 2 * 2 * kRows * 4;  // 231,616 B of the 232,448 B limit
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void st_shared_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_shared_u16(uint32_t a, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
__device__ __forceinline__ uint16_t ld_shared_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
// bf16 bits of x rounded toward +inf (-inf stays -inf), and back.
__device__ __forceinline__ uint16_t bf16_bits_ru(float x) { return __bfloat16_as_ushort(__float2bfloat16_ru(x)); }
__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) { return __bfloat162float(__ushort_as_bfloat16(b)); }
__device__ __forceinline__ float ld_shared_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gmem));
}

// K-major 128B-swizzled [2 halves][128 rows][128 B] tile: 16-byte chunk c
// (0..15) of row r.
__device__ __forceinline__ uint32_t tile_addr(uint32_t base, int r, int c) {
  return base + (c >> 3) * kHalfBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

// Packed fp32x2 arithmetic (FFMA2 / FADD2: two lanes per FMA-pipe issue).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n"
      " mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rc, {%6, %7};\n"
      " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n"
      " mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA pipe (packed fp32x2): round-to-nearest split
// through the 1.5*2^23 magic constant (the integer lands in the low mantissa
// bits and is shifted into the exponent), degree-5 polynomial on [-0.5, 0.5]
// (weighted least-squares fit, max relative error 2.4e-7 in fp32 Horner form —
// the MUFU ex2's level, so the bf16 rounding of P flips no more often than
// with ex2.approx; a cubic (2.1e-4) flipped ~2 % of the P values it produced).
// Inputs are clamped at -126 (-inf -> 2^-126).
#ifndef LP_EXP_POLY_DEG
#define LP_EXP_POLY_DEG 5
#endif
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f;
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 u = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = ffma2(u, make_float2(-1.f, -1.f), x);
#if LP_EXP_POLY_DEG == 4  // max relative error 2.6e-6
  float2 p = ffma2(make_float2(0.009570376f, 0.009570376f), f, make_float2(0.055918723f, 0.055918723f));
  p = ffma2(p, f, make_float2(0.24024746f, 0.24024746f));
  p = ffma2(p, f, make_float2(0.69312167f, 0.69312167f));
  p = ffma2(p, f, make_float2(0.99999928f, 0.99999928f));
#elif LP_EXP_POLY_DEG == 3  // 7.5e-5
  float2 p = ffma2(make_float2(0.055174146f, 0.055174146f), f, make_float2(0.24261758f, 0.24261758f));
  p = ffma2(p, f, make_float2(0.69326109f, 0.69326109f));
  p = ffma2(p, f, make_float2(0.99992758f, 0.99992758f));
#else
  float2 p = ffma2(make_float2(0.0013276408f, 0.0013276408f), f, make_float2(0.0096755205f, 0.0096755205f));
  p = ffma2(p, f, make_float2(0.055507131f, 0.055507131f));
  p = ffma2(p, f, make_float2(0.24022120f, 0.24022120f));
  p = ffma2(p, f, make_float2(0.69314694f, 0.69314694f));
  p = ffma2(p, f, make_float2(1.0000001f, 1.0000001f));
#endif
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Row max of a thread's slice: three-input max, two independent chains.
template <int N>
__device__ __forceinline__ float slice_max(const float (&v)[N]) {
  float a = -INFINITY, b = -INFINITY;
#pragma unroll
  for (int k = 0; k < N; k += 4) {
    a = fmax3(a, v[k], v[k + 1]);
    b = fmax3(b, v[k + 2], v[k + 3]);
  }
  return fmaxf(a, b);
}

// Softmax numerators of a thread's slice in place, 2^(s * scale - m), and
// their sum. The scale, the sum and the FMA-pipe exponentials run packed
// (fp32x2); pair q = (2q, 2q+1) goes to the polynomial iff q % kExpPairMod <
// kExpPairCnt, the rest to MUFU ex2 (the step is bound by FMA-pipe issue
// and MUFU throughput together; profiles/r02_attn_experiments.md).
#ifndef LP_EXP_PAIR_MOD
#define LP_EXP_PAIR_MOD 8
#define LP_EXP_PAIR_CNT 3
#endif
constexpr int kExpPairMod = LP_EXP_PAIR_MOD, kExpPairCnt = LP_EXP_PAIR_CNT;
template <int N>
__device__ __forceinline__ float slice_exp_sum(float (&v)[N], float scale, float m_use) {
  const float2 sc2 = make_float2(scale, scale), mm2 = make_float2(-m_use, -m_use);
  float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < N / 2; ++q) {
    const float2 x = ffma2(make_float2(v[2 * q], v[2 * q + 1]), sc2, mm2);
    float2 e;
    if (q % kExpPairMod < kExpPairCnt) {
      e = ex2_poly2(x);
    } else {
      e.x = ex2_ftz(x.x);
      e.y = ex2_ftz(x.y);
    }
    v[2 * q] = e.x;
    v[2 * q + 1] = e.y;
    if (q & 1) s1 = fadd2(s1, e);
    else s0 = fadd2(s0, e);
  }
  const float2 s = fadd2(s0, s1);
  return s.x + s.y;
}

// Diagnostic build only (-DLP_ATTN_PROF, scripts/attn_prof.py): clock64
// stamps per step for the MMA issuer, one softmax warp and the K producer of
// the first kProfCtas CTAs of KV head 0. Compiled out of the product library.
#ifdef LP_ATTN_PROF
constexpr int kProfCtas = 128, kProfSteps = 64;
__device__ unsigned long long g_attn_prof[kProfCtas][3][kProfSteps][8];
#define ATTN_PROF(role, step, ev)                                                            \
  do {                                                                                       \
    if (blockIdx.y == 0 && blockIdx.x < kProfCtas && (step) < kProfSteps && (step) >= 0)     \
      g_attn_prof[blockIdx.x][role][step][ev] = clock64();                                   \
  } while (0)
#else
#define ATTN_PROF(role, step, ev) \
  do {                            \
  } while (0)
#endif

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap kvm, const AttnCtx c) {
  KTL_SCOPE(kKtlAttnTc, 0);
  // The dynamic window must start 1024-byte aligned (128B-swizzle atoms);
  // trap loudly if it ever does not.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TcSmem::kBars);
  // K and V have separate rings: K(s) is released as soon as S(s) retires,
  // so the load of K(s+2) overlaps softmax(s) and PV(s); V(s) after PV(s).
  uint64_t* k_full = bars + 18;    // [3]
  uint64_t* k_empty = bars + 21;   // [3]
  uint64_t* s_full = bars + 4;     // [2]
  uint64_t* s_empty = bars + 6;    // [2]
  uint64_t* p_ready = bars + 8;    // [2] P buffer written (8 softmax warps)
  uint64_t* q_ready = bars + 10;
  uint64_t* p_free = bars + 24;    // [2] the PV that read the P buffer retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  uint64_t* v_full = bars + 26;    // [3]
  uint64_t* v_empty = bars + 29;   // [3]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  pdl_trigger();
  const int wi = blockIdx.x;
  const bool live = wi < *c.n_work;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kSoftmaxWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_ready[i], kSoftmaxWarps);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(q_ready, kSoftmaxWarps);
    fence_mbar_init();
  }
  if (warp == 1 && live) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (!live) {
    pdl_wait();
    return;
  }
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  const int g = blockIdx.y;
  const int G = c.nq / c.nkv;
  const int4 wk = c.work[wi];
  const int r = wk.x & 0xFFFF, row0 = wk.y;  // high bits: combine entry of a split item
  const int L = c.q_len[r], H = c.hist[r], qs = c.q_start[r];
  const int rows_total = L * G;
  const int* pages = c.page_list + c.page_off[r];
  const size_t ld_q = static_cast<size_t>(c.nq) * kD;
  const int row_hi = min(row0 + kRows - 1, rows_total - 1);
  const int p_hi = H + row_hi / G;
  const bool partial = wk.w >= 0;
  const int t_begin = wk.z;                               // first page
  const int t_end = partial ? wk.w : (p_hi + 1 + 63) / 64;  // one past the last page
  const int n_steps = (t_end - t_begin + 1) / 2;

  const uint32_t sQ = smem_u32(smem + TcSmem::kQ);
  const uint32_t sK = smem_u32(smem + TcSmem::kK), sV = smem_u32(smem + TcSmem::kV);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    // lane 0 streams K pages, lane 1 V pages (each into its own 3-stage ring).
    if (lane < 2) {
      const bool is_v = lane == 1;
      uint64_t* full = is_v ? v_full : k_full;
      uint64_t* empty = is_v ? v_empty : k_empty;
      uint8_t* ring = smem + (is_v ? TcSmem::kV : TcSmem::kK);
      const int ns = is_v ? kVStages : kKStages;
      for (int s = 0; s < n_steps; ++s) {
        const int st = s % ns;
        if (!is_v) ATTN_PROF(2, s, 0);
        mbar_wait(&empty[st], ((s / ns) & 1) ^ 1);
        if (!is_v) ATTN_PROF(2, s, 1);
        mbar_arrive_expect_tx(&full[st], kQBytes);
        const int t0 = t_begin + 2 * s;
        // A missing second page re-loads the first (finite values, masked).
        const int pg[2] = {pages[t0], t0 + 1 < t_end ? pages[t0 + 1] : pages[t0]};
#pragma unroll
        for (int pi = 0; pi < 2; ++pi) {
          const int plane = c.kv_plane0 + pg[pi] * 2 * c.nkv + g + (is_v ? c.nkv : 0);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d(ring + st * kQBytes + hf * kHalfBytes + pi * 64 * 128, &kvm, &full[st], hf * 64, 0, plane);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_o = idesc_bf16(kRows, kD) | (1u << 16);  // B (V) is MN-major
    const uint32_t t_o = tmem + 2 * kKeys;
    const uint32_t t_p = tmem + 3 * kKeys;  // P[2]: 128 keys as 64 packed bf16x2 columns each
    mbar_wait(q_ready, 0);
    tc_fence_after();
    auto issue_s = [&](int s) {
      const int st = s & 1;
      const int kst = s % kKStages;
      mbar_wait(&k_full[kst], (s / kKStages) & 1);
      if (s >= 2) mbar_wait(&s_empty[st], ((s >> 1) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t off = (k >> 2) * kHalfBytes + (k & 3) * 32;
          tc_mma_bf16(tmem + st * kKeys, sdesc_sw128(sQ + off), sdesc_sw128(sK + kst * kQBytes + off), idesc_s,
                      k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        tc_commit(&k_empty[kst]);
      }
      __syncwarp();
    };
    // S runs two steps ahead of PV: S(s+2) is queued right behind PV(s).
    if (n_steps > 0) issue_s(0);
    if (n_steps > 1) issue_s(1);
    for (int s = 0; s < n_steps; ++s) {
      const int st = s & 1;
      if (lane == 0) ATTN_PROF(0, s, 0);
      mbar_wait(&p_ready[st], (s >> 1) & 1);
      if (lane == 0) ATTN_PROF(0, s, 1);
      const int vst = s % kVStages;
      mbar_wait(&v_full[vst], (s / kVStages) & 1);
      if (lane == 0) ATTN_PROF(0, s, 2);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          // P (A operand) straight from TMEM: 16 keys = 8 packed bf16x2 columns per MMA.
          const uint64_t b = sdesc_sw128_mn(sV + vst * kQBytes + k * 16 * 128, kHalfBytes, 1024);
          tc_mma_bf16_ts(t_o, t_p + st * 64 + k * 8, b, idesc_o, (s > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(&p_free[st]);
        tc_commit(&v_empty[vst]);
      }
      __syncwarp();
      if (s + 2 < n_steps) issue_s(s + 2);
      if (lane == 0) ATTN_PROF(0, s, 3);
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;           // 0: columns 0-63, 1: columns 64-127
    const int rt = q4 * 32 + lane;             // tile row == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const int row = min(row0 + rt, rows_total - 1);
    const int j = row / G, hq = g * G + row % G;
    const int pos = H + j;
    const uint32_t red = smem_u32(smem + TcSmem::kRed);    // float [parity][grp][row]
    const int bar_id = 1 + q4;                 // the two warps sharing this lane quarter
    auto pair_sync = [&] { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    // This thread's half of the Q row -> smem (swizzled), once.
    const __nv_bfloat16* qrow = c.q + (qs + j) * ld_q + hq * kD;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) cp_async16(tile_addr(sQ, rt, grp * 8 + ch), qrow + (grp * 8 + ch) * 8);
    asm volatile("cp.async.wait_all;" ::: "memory");
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(q_ready);

    constexpr int kHalf = kKeys / 2;
    float m_run = -INFINITY, l_run = 0.f;  // l_run: this thread's columns only
    for (int s = 0; s < n_steps; ++s) {
      const int st = s & 1;
      const bool prof_me = warp == 2 && lane == 0;
      if (prof_me) ATTN_PROF(1, s, 0);
      mbar_wait(&s_full[st], (s >> 1) & 1);
      if (prof_me) ATTN_PROF(1, s, 1);
      tc_fence_after();
      float sc[kHalf];
#pragma unroll
      for (int cc = 0; cc < kHalf / 16; ++cc)
        tmem_ld16(tmem + lane_off + st * kKeys + grp * kHalf + cc * 16, sc + cc * 16);
      if (prof_me) ATTN_PROF(1, s, 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);  // S buffer may be overwritten

      const int kbase = (t_begin + 2 * s) * 64 + grp * kHalf;
      const int kvalid = min(kKeys, (t_end - t_begin - 2 * s) * 64) - grp * kHalf;  // keys of real pages
      if (!(kvalid >= kHalf && kbase + kHalf - 1 <= pos)) {  // a whole visible half needs no mask (long histories)
#pragma unroll
        for (int k = 0; k < kHalf; ++k)
          if (k >= kvalid || kbase + k > pos) sc[k] = -INFINITY;
      }
      float mx = slice_max(sc);
      const uint32_t rb = red + (s & 1) * 2 * kRows * 4;
      st_shared_f32(rb + (grp * kRows + rt) * 4, mx);
      pair_sync();
      mx = fmaxf(mx, ld_shared_f32(rb + ((grp ^ 1) * kRows + rt) * 4));
      if (prof_me) ATTN_PROF(1, s, 5);
      const float m_cand = fmaxf(m_run, mx * c.scale_log2);
      // Lazy rescale: keep the reference max unless the row max outgrew it.
      const bool grow = m_cand > m_run + kRescaleTau || (m_run == -INFINITY && m_cand != -INFINITY);
      const float m_new = grow ? m_cand : m_run;
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      const float corr = grow ? exp2f(m_run - m_use) : 1.f;
      m_run = m_new;
      // ex2.approx.ftz (MUFU) for most elements: exp2f adds a range check and
      // two conditional scalings per element; arguments here are <=
      // kRescaleTau and results below 2^-126 are negligible against the row
      // sum. 3 pairs in 8 run the polynomial on the FMA pipe (slice_exp_sum).
      const float sum = slice_exp_sum(sc, c.scale_log2, m_use);
      l_run = l_run * corr + sum;
      if (prof_me) ATTN_PROF(1, s, 2);

      // P buffer s&1 was read by PV(s-2); O may be rescaled only after every
      // issued PV (up to s-1) retired (PVs retire in order).
      if (s >= 2) {
        mbar_wait(&p_free[s & 1], ((s >> 1) & 1) ^ 1);
        tc_fence_after();
      }
      if (s > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
        mbar_wait(&p_free[(s - 1) & 1], ((s - 1) >> 1) & 1);
        tc_fence_after();
        {
          const uint32_t t_o = tmem + lane_off + 2 * kKeys + grp * (kD / 2);
#pragma unroll 1
          for (int cc = 0; cc < kD / 32; ++cc) {
            float o[16];
            tmem_ld16(t_o + cc * 16, o);
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= corr;
            tmem_st16(t_o + cc * 16, o);
          }
          tc_wait_st();
        }
      }
      if (prof_me) ATTN_PROF(1, s, 6);
      // P half-row (bf16 pairs) -> TMEM columns [grp*32, grp*32+32) of the P
      // region (the PV MMA reads A from tensor memory: no smem round trip, no
      // async-proxy fence).
      {
        const uint32_t t_pw = tmem + lane_off + 3 * kKeys + (s & 1) * 64 + grp * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = __uint_as_float(pack_bf16x2(sc[h * 32 + 2 * i], sc[h * 32 + 2 * i + 1]));
          tmem_st16(t_pw + h * 16, w);
        }
        tc_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_ready[s & 1]);
      if (prof_me) ATTN_PROF(1, s, 3);
    }

    // Epilogue: O row / l, l = both groups' partial sums (same reference max).
    // (the parity buffer of step n_steps was last read before step n_steps-1's barrier)
    const uint32_t lsum = red + (n_steps & 1) * 2 * kRows * 4;
    st_shared_f32(lsum + (grp * kRows + rt) * 4, l_run);
    pair_sync();
    const float l_tot = l_run + ld_shared_f32(lsum + ((grp ^ 1) * kRows + rt) * 4);
    if (n_steps > 0) {  // the last PV retired
      mbar_wait(&p_free[(n_steps - 1) & 1], ((n_steps - 1) >> 1) & 1);
      tc_fence_after();
    }
    const uint32_t t_o = tmem + lane_off + 2 * kKeys + grp * (kD / 2);
    if (!partial) {
      const float inv = 1.f / l_tot;
      __nv_bfloat16* dst = c.out + (qs + j) * ld_q + hq * kD + grp * (kD / 2);
#pragma unroll 1
      for (int cc = 0; cc < kD / 32; ++cc) {
        float o[16];
        tmem_ld16(t_o + cc * 16, o);
        if (row0 + rt < rows_total) {
          uint4 w[2];
          uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int i = 0; i < 8; ++i) wp[i] = pack_bf16x2(o[2 * i] * inv, o[2 * i + 1] * inv);
          reinterpret_cast<uint4*>(dst + cc * 16)[0] = w[0];
          reinterpret_cast<uint4*>(dst + cc * 16)[1] = w[1];
        }
      }
    } else {
      const size_t slab = static_cast<size_t>(wi) * c.nkv + g;
      float* dst = c.ws_o + (slab * kRows + rt) * kD + grp * (kD / 2);
#pragma unroll 1
      for (int cc = 0; cc < kD / 32; ++cc) {
        float o[16];
        tmem_ld16(t_o + cc * 16, o);
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(dst + cc * 16 + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
      }
      if (grp == 0) {
        c.ws_ml[(slab * kRows + rt) * 2 + 0] = m_run;
        c.ws_ml[(slab * kRows + rt) * 2 + 1] = l_tot;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  // Key split: the last split of this row block to finish merges it (the
  // exchange buffer is free once every softmax warp is past the barrier).
  if (partial) attn_merge_if_last<128>(c, wi, g, kThreads / 32, reinterpret_cast<int*>(smem + TcSmem::kRed));
}


// ---------------------------------------------------------------------------
// Persistent variant. The one-CTA-per-work-item grid leaves SMs idle when the
// item count is not a multiple of the SM count (7B 512-token chunk: 112 CTAs
// for 148 SMs; 32B: 160 CTAs = 1.08 waves) and pays the CTA prologue (TMEM
// allocation, barrier init, pipeline ramp) per item. Here one CTA per SM walks
// a host-built list of pieces — (128-row block, kv head, page range) — cut
// so every list costs the same (executor.cu, McNaughton's rule); the TMA
// rings, S/P buffers and their barrier phases run on one global step counter
// across pieces (the producer streams the next piece's keys while the current
// one drains), the Q tile is reloaded per piece once the previous piece's
// MMAs retired, and a unit split across two lists is merged by its
// last-finishing piece from fp32 partials.
constexpr int kPKStages = 3;
constexpr int kPVStages = 3;
// Softmax groups of the persistent kernel (column slices of every step):
// 4 groups (16 softmax warps, 32 keys each) halve each thread's work per
// step but measured 2 % slower than 2 (profiles/r02_attn_experiments.md).
#ifndef LP_ATTN_SOFT_GROUPS
#define LP_ATTN_SOFT_GROUPS 2
#endif
constexpr int kTcpGroups = LP_ATTN_SOFT_GROUPS;
static_assert(kTcpGroups == 2 || kTcpGroups == 4, "softmax groups: 2 or 4");
constexpr int kTcpSoftWarps = 4 * kTcpGroups;
constexpr int kTcpThreads = 64 + 32 * kTcpSoftWarps;

struct TcpSmem {
  static constexpr int kQ = 0;                                  // [32 KiB]
  static constexpr int kK = kQ + kQBytes;                       // [3][32 KiB]
  static constexpr int kV = kK + kPKStages * kQBytes;           // [3][32 KiB]
  static constexpr int kBars = kV + kPVStages * kQBytes;
  static constexpr int kRed = kBars + 256;  // [2 parity][groups][128 rows]: fp32 for 2 groups, bf16 for 4
  static constexpr int kTotal = kRed + 2 * 2 * kRows * 4;       // 231,680 B of the 232,448 B limit
};

struct Piece {
  int r, row0, t_begin, t_end, g, ci, slot;
};
__device__ __forceinline__ Piece load_piece(const AttnCtx& c, int i) {
  const int4 a = c.work[i], b = c.work2[i];
  return Piece{a.x, a.y, a.z, a.w, b.x, b.y, b.z};
}

__global__ void __launch_bounds__(kTcpThreads, 1)
    attn_tcp_kernel(const __grid_constant__ CUtensorMap kvm, const AttnCtx c) {
  KTL_SCOPE(kKtlAttnTcp, 0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TcpSmem::kBars);
  uint64_t* k_full = bars + 0;     // [3]
  uint64_t* k_empty = bars + 3;    // [3]
  uint64_t* v_full = bars + 6;     // [3]
  uint64_t* v_empty = bars + 9;    // [3]
  uint64_t* s_full = bars + 12;    // [2]
  uint64_t* s_empty = bars + 14;   // [2]
  uint64_t* p_ready = bars + 16;   // [2]
  uint64_t* p_free = bars + 18;    // [2]
  uint64_t* q_ready = bars + 20;   // Q tile of piece j landed (phase j)
  uint64_t* q_free = bars + 21;    // every MMA of piece j retired (the Q tile may be replaced)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
  int* s_flag = reinterpret_cast<int*>(bars + 23);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  pdl_trigger();
  const int p_beg = c.cta_off[blockIdx.x], p_end = c.cta_off[blockIdx.x + 1];
  const bool live = p_end > p_beg;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kPKStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kPVStages; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], kTcpSoftWarps);
      mbar_init(&p_ready[i], kTcpSoftWarps);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(q_ready, kTcpSoftWarps);
    mbar_init(q_free, 1);
    fence_mbar_init();
  }
  if (warp == 1 && live) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  if (!live) return;
  const uint32_t tmem = *tmem_slot;
  const int G = c.nq / c.nkv;
  const size_t ld_q = static_cast<size_t>(c.nq) * kD;
  const uint32_t sQ = smem_u32(smem + TcpSmem::kQ);
  const uint32_t sK = smem_u32(smem + TcpSmem::kK), sV = smem_u32(smem + TcpSmem::kV);
  auto steps_of = [](const Piece& p) { return (p.t_end - p.t_begin + 1) / 2; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    if (lane < 2) {
      const bool is_v = lane == 1;
      uint64_t* full = is_v ? v_full : k_full;
      uint64_t* empty = is_v ? v_empty : k_empty;
      uint8_t* ring = smem + (is_v ? TcpSmem::kV : TcpSmem::kK);
      const int ns = is_v ? kPVStages : kPKStages;
      int gs = 0;
      for (int i = p_beg; i < p_end; ++i) {
        const Piece pc = load_piece(c, i);
        const int* pages = c.page_list + c.page_off[pc.r];
        const int n = steps_of(pc);
        for (int s = 0; s < n; ++s, ++gs) {
          const int st = gs % ns;
          mbar_wait(&empty[st], ((gs / ns) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], kQBytes);
          const int t0 = pc.t_begin + 2 * s;
          const int pg[2] = {pages[t0], t0 + 1 < pc.t_end ? pages[t0 + 1] : pages[t0]};
#pragma unroll
          for (int pi = 0; pi < 2; ++pi) {
            const int plane = c.kv_plane0 + pg[pi] * 2 * c.nkv + pc.g + (is_v ? c.nkv : 0);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d(ring + st * kQBytes + hf * kHalfBytes + pi * 64 * 128, &kvm, &full[st], hf * 64, 0,
                          plane);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(kRows, kKeys);
    constexpr uint32_t idesc_o = idesc_bf16(kRows, kD) | (1u << 16);  // B (V) is MN-major
    const uint32_t t_o = tmem + 2 * kKeys;
    const uint32_t t_p = tmem + 3 * kKeys;
    int gs = 0;
    for (int i = p_beg, j = 0; i < p_end; ++i, ++j) {
      const Piece pc = load_piece(c, i);
      const int n = steps_of(pc);
      const uint32_t q_tile = sQ;
      mbar_wait(q_ready, j & 1);
      tc_fence_after();
      auto issue_s = [&](int x) {  // global step x of this piece
        const int st = x & 1, kst = x % kPKStages;
        mbar_wait(&k_full[kst], (x / kPKStages) & 1);
        if (x >= 2) mbar_wait(&s_empty[st], ((x >> 1) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalfBytes + (k & 3) * 32;
            tc_mma_bf16(tmem + st * kKeys, sdesc_sw128(q_tile + off), sdesc_sw128(sK + kst * kQBytes + off), idesc_s,
                        k > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[st]);
          tc_commit(&k_empty[kst]);
        }
        __syncwarp();
      };
      if (n > 0) issue_s(gs);
      if (n > 1) issue_s(gs + 1);
      for (int s = 0; s < n; ++s) {
        const int x = gs + s, st = x & 1, vst = x % kPVStages;
        mbar_wait(&p_ready[st], (x >> 1) & 1);
        mbar_wait(&v_full[vst], (x / kPVStages) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kKeys / 16; ++k) {
            const uint64_t b = sdesc_sw128_mn(sV + vst * kQBytes + k * 16 * 128, kHalfBytes, 1024);
            tc_mma_bf16_ts(t_o, t_p + st * 64 + k * 8, b, idesc_o, (s > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&p_free[st]);
          tc_commit(&v_empty[vst]);
        }
        __syncwarp();
        if (s + 2 < n) issue_s(x + 2);
      }
      if (elect_one()) tc_commit(q_free);  // this piece's MMAs retired: the Q tile may be replaced
      __syncwarp();
      gs += n;
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // kTcpGroups softmax groups of 4 warps; group grp owns key columns
    // [grp*kSlice, (grp+1)*kSlice) of every step and D columns
    // [grp*kD/kG, ...) of O. The warps sharing a TMEM lane quarter (one per
    // group) exchange row maxima through shared memory.
    constexpr int kG = kTcpGroups;
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int rt = q4 * 32 + lane;
    const int stid = threadIdx.x - 64;         // 0..128*kG-1 among the softmax threads
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t red = smem_u32(smem + TcpSmem::kRed);
    const int bar_id = 1 + q4;
    auto pair_sync = [&] { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(32 * kG) : "memory"); };
    auto soft_sync = [&] { asm volatile("bar.sync 9, %0;" ::"n"(128 * kG) : "memory"); };
    constexpr int kHalf = kKeys / kG;          // key columns per group per step
    constexpr int kDg = kD / kG;               // O columns per group
    int gs = 0;
    for (int i = p_beg, jj = 0; i < p_end; ++i, ++jj) {
      const Piece pc = load_piece(c, i);
      const int n = steps_of(pc);
      const int L = c.q_len[pc.r], H = c.hist[pc.r], qs = c.q_start[pc.r];
      const int rows_total = L * G;
      const int row = min(pc.row0 + rt, rows_total - 1);
      const int j = row / G, hq = pc.g * G + row % G;
      const int pos = H + j;
      // Q tile of this piece (the previous piece's MMAs have retired).
      const uint32_t q_tile = sQ;
      if (jj >= 1) mbar_wait(q_free, (jj - 1) & 1);
      const __nv_bfloat16* qrow = c.q + (qs + j) * ld_q + hq * kD;
#pragma unroll
      for (int ch = 0; ch < 16 / kG; ++ch)
        cp_async16(tile_addr(q_tile, rt, grp * (16 / kG) + ch), qrow + (grp * (16 / kG) + ch) * 8);
      asm volatile("cp.async.wait_all;" ::: "memory");
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);

      float m_run = -INFINITY, l_run = 0.f;
      for (int s = 0; s < n; ++s) {
        const int x = gs + s, st = x & 1;
        mbar_wait(&s_full[st], (x >> 1) & 1);
        tc_fence_after();
        float sc[kHalf];
        {  // all four S loads in flight before the first wait
          uint32_t r[kHalf / 16][16];
#pragma unroll
          for (int cc = 0; cc < kHalf / 16; ++cc) tmem_ld16_issue(tmem + lane_off + st * kKeys + grp * kHalf + cc * 16, r[cc]);
#pragma unroll
          for (int cc = 0; cc < kHalf / 16; ++cc) {
            tmem_ld16_wait(r[cc]);
#pragma unroll
            for (int q = 0; q < 16; ++q) sc[cc * 16 + q] = __uint_as_float(r[cc][q]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[st]);

        const int kbase = (pc.t_begin + 2 * s) * 64 + grp * kHalf;
        const int kvalid = min(kKeys, (pc.t_end - pc.t_begin - 2 * s) * 64) - grp * kHalf;
        if (!(kvalid >= kHalf && kbase + kHalf - 1 <= pos)) {
#pragma unroll
          for (int k = 0; k < kHalf; ++k)
            if (k >= kvalid || kbase + k > pos) sc[k] = -INFINITY;
        }
        float mx = slice_max(sc);
        if constexpr (kG == 2) {
          const uint32_t rb = red + (x & 1) * 2 * kRows * 4;
          st_shared_f32(rb + (grp * kRows + rt) * 4, mx);
          pair_sync();
          mx = fmaxf(mx, ld_shared_f32(rb + ((grp ^ 1) * kRows + rt) * 4));
        } else {
          // bf16 rounded up (the exchange buffer holds 2 parities x kG groups
          // x 128 rows in 2 KiB): every thread of a row takes the max of the
          // same kG rounded values, so the reference max stays consistent;
          // it only has to bound the row (lazy rescale tolerates 2^tau).
          const uint32_t rb = red + (x & 1) * kG * kRows * 2;
          st_shared_u16(rb + (grp * kRows + rt) * 2, bf16_bits_ru(mx));
          pair_sync();
          mx = -INFINITY;
#pragma unroll
          for (int g2 = 0; g2 < kG; ++g2) mx = fmaxf(mx, bf16_bits_to_f32(ld_shared_u16(rb + (g2 * kRows + rt) * 2)));
        }
        const float m_cand = fmaxf(m_run, mx * c.scale_log2);
        const bool grow = m_cand > m_run + kRescaleTau || (m_run == -INFINITY && m_cand != -INFINITY);
        const float m_new = grow ? m_cand : m_run;
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float corr = grow ? exp2f(m_run - m_use) : 1.f;
        m_run = m_new;
        const float sum = slice_exp_sum(sc, c.scale_log2, m_use);
        l_run = l_run * corr + sum;
        if (x >= 2) {  // P buffer st was read by PV(x - 2)
          mbar_wait(&p_free[st], ((x >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        if (s > 0 && __any_sync(0xffffffffu, corr != 1.f)) {  // O holds this piece's PVs up to s - 1
          mbar_wait(&p_free[(x - 1) & 1], ((x - 1) >> 1) & 1);
          tc_fence_after();
          const uint32_t t_o = tmem + lane_off + 2 * kKeys + grp * kDg;
#pragma unroll 1
          for (int cc = 0; cc < kDg / 16; ++cc) {
            float o[16];
            tmem_ld16(t_o + cc * 16, o);
#pragma unroll
            for (int q = 0; q < 16; ++q) o[q] *= corr;
            tmem_st16(t_o + cc * 16, o);
          }
          tc_wait_st();
        }
        {
          const uint32_t t_pw = tmem + lane_off + 3 * kKeys + st * 64 + grp * (kHalf / 2);
#pragma unroll
          for (int h = 0; h < kHalf / 32; ++h) {
            float w[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) w[q] = __uint_as_float(pack_bf16x2(sc[h * 32 + 2 * q], sc[h * 32 + 2 * q + 1]));
            tmem_st16(t_pw + h * 16, w);
          }
          tc_wait_st();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[st]);
      }

      // Epilogue of the piece: row sum over both column halves, then O / l
      // (bf16) or the fp32 partial of a split unit.
      const int xe = gs + n;  // the next step's exchange parity is free of this piece's max exchange
      float l_tot;
      if constexpr (kG == 2) {
        const uint32_t lsum = red + (xe & 1) * 2 * kRows * 4;
        st_shared_f32(lsum + (grp * kRows + rt) * 4, l_run);
        pair_sync();
        l_tot = l_run + ld_shared_f32(lsum + ((grp ^ 1) * kRows + rt) * 4);
        pair_sync();  // the next piece's first step writes this parity again
      } else {
        // The fp32 row sums need the whole exchange buffer: every softmax
        // warp is past its last max exchange before it is overwritten, and
        // every sum is read before the next piece's first exchange.
        soft_sync();
        st_shared_f32(red + (grp * kRows + rt) * 4, l_run);
        pair_sync();
        l_tot = 0.f;
#pragma unroll
        for (int g2 = 0; g2 < kG; ++g2) l_tot += ld_shared_f32(red + (g2 * kRows + rt) * 4);
        soft_sync();
      }
      if (n > 0) {
        mbar_wait(&p_free[(xe - 1) & 1], ((xe - 1) >> 1) & 1);
        tc_fence_after();
      }
      const uint32_t t_o = tmem + lane_off + 2 * kKeys + grp * kDg;
      if (pc.ci < 0) {
        const float inv = 1.f / l_tot;
        __nv_bfloat16* dst = c.out + (qs + j) * ld_q + hq * kD + grp * kDg;
#pragma unroll 1
        for (int cc = 0; cc < kDg / 16; ++cc) {
          float o[16];
          tmem_ld16(t_o + cc * 16, o);
          if (pc.row0 + rt < rows_total) {
            uint4 w[2];
            uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
            for (int q = 0; q < 8; ++q) wp[q] = pack_bf16x2(o[2 * q] * inv, o[2 * q + 1] * inv);
            reinterpret_cast<uint4*>(dst + cc * 16)[0] = w[0];
            reinterpret_cast<uint4*>(dst + cc * 16)[1] = w[1];
          }
        }
        tc_fence_before();
      } else {
        float* dst = c.ws_o + (static_cast<size_t>(pc.slot) * kRows + rt) * kD + grp * kDg;
#pragma unroll 1
        for (int cc = 0; cc < kDg / 16; ++cc) {
          float o[16];
          tmem_ld16(t_o + cc * 16, o);
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            *reinterpret_cast<float4*>(dst + cc * 16 + q) = make_float4(o[q], o[q + 1], o[q + 2], o[q + 3]);
        }
        tc_fence_before();
        if (grp == 0) {
          c.ws_ml[(static_cast<size_t>(pc.slot) * kRows + rt) * 2 + 0] = m_run;
          c.ws_ml[(static_cast<size_t>(pc.slot) * kRows + rt) * 2 + 1] = l_tot;
        }
        // The unit's last piece to finish merges every piece's partial.
        __threadfence();
        soft_sync();
        if (stid == 0) {
          const int4 e = c.combine[pc.ci];
          int* cnt = c.comb_cnt + pc.ci;
          const int last = atomicAdd(cnt, 1) == e.w - 1;
          if (last) *cnt = 0;
          *s_flag = last;
        }
        soft_sync();
        if (*s_flag) {
          __threadfence();
          const int4 e = c.combine[pc.ci];
          const int first = e.z, np = e.w;
          for (int it = stid; it < kRows * (kD / 16); it += 128 * kG) {
            const int rl = it / (kD / 16), qc = it % (kD / 16);
            const int mrow = pc.row0 + rl;
            if (mrow >= rows_total) continue;
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.f;
            float m_all = -INFINITY;
            for (int k = 0; k < np; ++k)
              m_all = fmaxf(m_all, __ldcg(c.ws_ml + (static_cast<size_t>(first + k) * kRows + rl) * 2));
            float l_all = 0.f;
            for (int k = 0; k < np; ++k) {
              const size_t sb = static_cast<size_t>(first + k) * kRows + rl;
              const float mk = __ldcg(c.ws_ml + sb * 2), lk = __ldcg(c.ws_ml + sb * 2 + 1);
              const float wk = mk == -INFINITY ? 0.f : exp2f(mk - m_all);
              l_all += wk * lk;
              const float4* src = reinterpret_cast<const float4*>(c.ws_o + sb * kD + qc * 16);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                const float4 xv = __ldcg(src + v);
                acc[4 * v + 0] += wk * xv.x;
                acc[4 * v + 1] += wk * xv.y;
                acc[4 * v + 2] += wk * xv.z;
                acc[4 * v + 3] += wk * xv.w;
              }
            }
            const float inv = 1.f / l_all;
            const int mj = mrow / G, mh = pc.g * G + mrow % G;
            __nv_bfloat16* dst = c.out + (qs + mj) * ld_q + mh * kD + qc * 16;
            uint4 w[2];
            uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
            for (int q = 0; q < 8; ++q) wp[q] = pack_bf16x2(acc[2 * q] * inv, acc[2 * q + 1] * inv);
            reinterpret_cast<uint4*>(dst)[0] = w[0];
            reinterpret_cast<uint4*>(dst)[1] = w[1];
          }
        }
        soft_sync();  // s_flag is rewritten by the next split piece
      }
      gs += n;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


}  // namespace

void attention_prefill_tc(const AttnCtx& c, const CUtensorMap& kv_map, int work_cap, cudaStream_t st) {
  constexpr int smem = TcSmem::kTotal;
  smem_attr_once(reinterpret_cast<const void*>(attn_tc_kernel), smem);
  launch_k(attn_tc_kernel, dim3(work_cap, c.nkv), dim3(kThreads), smem, st, kv_map, c);
}

void attention_prefill_tc_persistent(const AttnCtx& c, const CUtensorMap& kv_map, int n_cta, cudaStream_t st) {
  constexpr int smem = TcpSmem::kTotal;

  smem_attr_once(reinterpret_cast<const void*>(attn_tcp_kernel), smem);
  launch_k(attn_tcp_kernel, dim3(n_cta), dim3(kTcpThreads), smem, st, kv_map, c);
}

#ifdef LP_ATTN_PROF
extern "C" int lp_debug_attn_prof(unsigned long long* out, size_t n) {
  const size_t bytes = std::min(n * sizeof(unsigned long long), sizeof(g_attn_prof));
  return cudaMemcpyFromSymbol(out, g_attn_prof, bytes) == cudaSuccess ? 0 : -1;
}
extern "C" int lp_debug_attn_prof_reset() {
  static unsigned long long zero[kProfCtas][3][kProfSteps][8];
  return cudaMemcpyToSymbol(g_attn_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace lp

KTL_EXPORT(attn_tc)
