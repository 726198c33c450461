// tcgen05 GEMM — see gemm_sm100.cuh for the orientation and roles.
//
// Two variants of one persistent, warp-specialised kernel:
//   kPair = 1 : one CTA per 128-row weight tile, tcgen05.mma.cta_group::1.
//   kPair = 2 : a CTA pair (cluster of 2) per 256-row weight tile,
//               tcgen05.mma.cta_group::2 issued by the leader CTA. Each CTA
//               TMA-loads its own 128 weight rows and HALF of the token tile,
//               so every activation byte crosses L2->SM once per 256 weight
//               rows (not per 128) and per-SM shared-memory operand traffic
//               halves. Used for token tiles of >= 128 columns.
#include <atomic>
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm_sm100.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace lp {

namespace {

constexpr int kBM = 128;            // weight rows per CTA (TMEM lanes)
constexpr int kBK = 64;             // K per stage: one 128-byte swizzle row of bf16
// Epilogue warp groups of 4 (each covers all 128 TMEM lanes, alternate
// 16-column chunks). Two groups halve the last tile's epilogue in isolation
// but cost ~1.5 % on whole bucket forwards (8 more warps polling barriers
// next to the TMA / MMA warps; profiles/r02_gemm_timeline.md), so one is built.
#ifndef LP_GEMM_EPI_GROUPS
#define LP_GEMM_EPI_GROUPS 1
#endif
constexpr int kEpiGroups = LP_GEMM_EPI_GROUPS;
constexpr int kThreads = 64 + 128 * kEpiGroups;  // warp0 TMA, warp1 MMA, then the epilogue groups
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kSmemBudget = 196 * 1024;
#ifndef LP_GEMM_MAX_STAGES
#define LP_GEMM_MAX_STAGES 8
#endif
constexpr int kMaxStages = LP_GEMM_MAX_STAGES;  // ring depth cap (narrow token tiles fit more)
// Epilogue staging, double-buffered per epilogue group: SiLU uses [16
// tokens][64 features] bf16 (both groups), the fused QKV/RoPE epilogue [128
// rows][17] fp32 (padded: conflict-free; group 0 only).
constexpr int kEpiStageBytes = 128 * 17 * 4;
constexpr int kEpiStage1Bytes = 16 * 64 * 2;

template <int BN, int kPair>
struct Cfg {
  static constexpr int kBRows = BN / kPair;       // token rows of B held by this CTA
  static constexpr int kABytes = kBM * kBK * 2;   // 16 KiB
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > kMaxStages ? kMaxStages : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmem = 1024 /*align*/ + kStages * kStageBytes + kBarBytes + 2 * kEpiStageBytes +
                               (kEpiGroups - 1) * 2 * kEpiStage1Bytes;
  static_assert(kSmem <= 227 * 1024, "GEMM shared memory over the per-CTA limit");
};

// x * sigmoid(x) with the fast exp / divide intrinsics (|rel err| ~ 1e-7,
// far below the bf16 rounding that follows).
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// Named barrier of one epilogue group (ids 1, 2; 128 threads each).
__device__ __forceinline__ void epi_bar(int group) { asm volatile("bar.sync %0, 128;" ::"r"(1 + group) : "memory"); }

// Diagnostic build only (-DLP_GEMM_PROF, scripts/gemm_prof.py): %globaltimer
// stamps of one launch's phases per CTA, recorded for the launch whose (M, K)
// matches g_gemm_prof_sel. Compiled out of the product library.
#ifdef LP_GEMM_PROF
constexpr int kProfCtas = 160, kProfEv = 12;
__device__ unsigned long long g_gemm_prof[kProfCtas][kProfEv];
__device__ int g_gemm_prof_sel[2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GEMM_PROF(ev)                                                                              \
  do {                                                                                             \
    if (args.M == g_gemm_prof_sel[0] && args.K == g_gemm_prof_sel[1] && blockIdx.x < kProfCtas) \
      g_gemm_prof[blockIdx.x][ev] = gtimer();                                                      \
  } while (0)
#else
#define GEMM_PROF(ev) \
  do {                \
  } while (0)
#endif

template <int BN, int kPair>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  KTL_SCOPE(kKtlGemm, args.M);
  using C = Cfg<BN, kPair>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __nv_bfloat16* epi_stage =
      reinterpret_cast<__nv_bfloat16*>(smem + C::kStages * C::kStageBytes + C::kBarBytes);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = kPair == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  if (threadIdx.x == 0) GEMM_PROF(0);  // entry
  pdl_trigger();

  // n_dev is written by the pre-graph H2D copy, never by a kernel: safe before pdl_wait.
  const int n_live = args.n_dev ? min(*args.n_dev, args.N) : args.N;
  if (n_live <= 0) {  // nothing live (e.g. an LM head no member wants): no loads, no MMAs
    pdl_wait();
    return;
  }
  const int m_tiles = args.M / (kBM * kPair);   // tiles of this variant (128 or 256 rows)
  // Token tiles are sized from the LIVE token count: ceil(n_live / BN) tiles
  // of equal width tw (a multiple of 16 <= BN), and each tile's MMA runs with
  // N = its live width rounded up to 16 (the instruction descriptor is a
  // runtime operand), so a graph captured for l_pad * depth tokens does no
  // tensor work for padding beyond the next multiple of 16.
  int n_tiles = max(1, (n_live + BN - 1) / BN);
  if (args.ntiles_dev) n_tiles = max(n_tiles, min(*args.ntiles_dev, (n_live + 15) / 16));
  const int tw = min(BN, ((n_live + n_tiles - 1) / n_tiles + 15) / 16 * 16);
  const int num_kb = args.K / kBK;
  // Split-K factor: from device metadata when the plan is chosen per batch (pre-graph H2D).
  const int split_raw = args.splits_dev ? *args.splits_dev : args.splits;
  const bool sk = split_raw < 0 && args.sk_tab != nullptr;  // stream-K
  const int splits = max(1, split_raw);
  const int units = splits * m_tiles * n_tiles;
  const int worker = blockIdx.x / kPair;        // CTA (pair) index
  const int n_workers = gridDim.x / kPair;
  // Stream-K over the (weight tile, K-block) space, m-major: the workers form
  // groups of one CTA (pair) per live token tile, group j owns steps
  // [j*per, min((j+1)*per, total)) and its members run them in lockstep on
  // their own token tiles, so every weight tile is fetched from DRAM once and
  // shared through L2 (as consecutive split-K units are). Workers beyond the
  // last whole group idle.
  const int sk_tiles_n = (n_live + tw - 1) / tw;
  const int sk_groups = max(1, n_workers / sk_tiles_n);
  const int sk_total = m_tiles * num_kb;
  const int sk_per = (sk_total + sk_groups - 1) / sk_groups;
  const int sk_group = worker / sk_tiles_n, sk_n = worker % sk_tiles_n;
  const int sk_beg = sk && sk_group < sk_groups ? min(sk_total, sk_group * sk_per) : 0;
  const int sk_end = sk && sk_group < sk_groups ? min(sk_total, sk_beg + sk_per) : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * kPair);  // every epilogue warp of the pair
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (kPair == 2) tmem_alloc_pair<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair == 2) cluster_sync();  // peer barriers initialised before remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GEMM_PROF(1);  // barriers, TMEM, cluster ready

  // MMA N of the tile starting at n0 (a multiple of 16, <= tw).
  auto mma_n = [&](int n0) { return min(tw, (n_live - n0 + 15) / 16 * 16); };
  // One accumulation this CTA (pair) runs: output tile (m0, n0), K-blocks
  // [kb0, kb1), written to ws slice s: split s (split-K) or, under stream-K,
  // segment seg of the tile's nseg.
  struct Seg { int s, m0, n0, kb0, kb1, seg, nseg, tile; };
  // Iterators: `it` = next unit (split-K) or next flattened position (stream-K).
  auto first_it = [&]() { return sk ? sk_beg : worker; };
  auto next_seg = [&](int& it, Seg& g) -> bool {
    if (sk) {
      if (it >= sk_end) return false;
      const int mt = it / num_kb;
      g.kb0 = it % num_kb;
      g.kb1 = min(num_kb, g.kb0 + (sk_end - it));
      const int t0 = mt * num_kb;
      g.seg = it / sk_per - t0 / sk_per;
      g.nseg = (t0 + num_kb - 1) / sk_per - t0 / sk_per + 1;
      it += g.kb1 - g.kb0;
      g.s = g.seg;  // segment j of a tile -> ws slice j
      g.tile = mt * sk_tiles_n + sk_n;
      g.m0 = mt * kBM * kPair + static_cast<int>(rank) * kBM;
      g.n0 = sk_n * tw;
      return true;
    }
    while (it < units) {
      const int w = it;
      it += n_workers;
      const int n = w % n_tiles;
      const int rest = w / n_tiles;
      const int m = rest % m_tiles;
      g.s = rest / m_tiles;
      g.m0 = m * kBM * kPair + static_cast<int>(rank) * kBM;  // this CTA's 128 weight rows
      g.n0 = n * tw;
      const int base = num_kb / splits, rem = num_kb % splits;
      g.kb0 = g.s * base + min(g.s, rem);
      g.kb1 = g.kb0 + base + (g.s < rem ? 1 : 0);
      g.seg = 0;
      g.nseg = 1;
      g.tile = w;
      if (g.n0 < n_live) return true;
    }
    return false;
  };

  if (warp == 0) {
    // ----------------------------------------------------------- TMA producer
    if (elect_one()) {
      // A weight tile with a single consumer streams once (evict first); with
      // several token tiles its sibling units (consecutive unit ids, resident
      // at the same time) re-read it from L2, so keep normal priority.
      const uint64_t pol_w = n_tiles > 1 ? policy_evict_normal() : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();   // activations are re-read per m tile
      const uint32_t bar0 = kPair == 2 ? mapa(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
      auto load = [&](int stage, int kb, int m0, int n0, bool a_part, bool b_part) {
        const uint32_t bar = bar0 + stage * 8;
        if constexpr (kPair == 2) {
          // The pair's MMA takes N/2 token rows from each CTA: rank r holds
          // tokens [n0 + r*N/2, n0 + (r+1)*N/2) at the top of its B stage.
          if (a_part) tma_load_2d_pair(sA + stage * C::kABytes, &tmA, bar, kb * kBK, m0, pol_w);
          if (b_part)
            tma_load_2d_pair(sB + stage * C::kBBytes, &tmB, bar, kb * kBK,
                             n0 + static_cast<int>(rank) * (mma_n(n0) / 2), pol_x);
        } else {
          if (a_part) tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * kBK, m0, pol_w);
          if (b_part) tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBK, n0, pol_x);
        }
      };
      // The leader's full barrier expects the bytes of the whole pair.
      auto expect = [&](int stage) {
        if (leader) mbar_arrive_expect_tx(&full[stage], C::kStageBytes * kPair);
      };
      // Weight tiles do not depend on the previous kernel: fill the pipeline
      // with them before waiting on it (PDL), then add the activation tiles.
      int it = first_it();
      Seg g;
      bool have = next_seg(it, g);
      const int pre = have ? min(g.kb1 - g.kb0, C::kStages) : 0;
      for (int i = 0; i < pre; ++i) {
        expect(i);
        load(i, g.kb0 + i, g.m0, g.n0, true, false);
      }
      pdl_wait();
      GEMM_PROF(2);  // predecessor done
      for (int i = 0; i < pre; ++i) load(i, g.kb0 + i, 0, g.n0, false, true);
      int stage = pre % C::kStages;
      uint32_t phase = pre == C::kStages ? 1u : 0u;
      for (int skip = pre; have; have = next_seg(it, g), skip = 0) {
        for (int kb = g.kb0 + skip; kb < g.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          expect(stage);
          load(stage, kb, g.m0, g.n0, true, true);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
      GEMM_PROF(3);  // last load issued
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer (leader of a pair)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      int it = first_it();
      Seg g;
#ifdef LP_GEMM_PROF
      int n_mma = 0;
#endif
      while (next_seg(it, g)) {
        const int kb0 = g.kb0, kb1 = g.kb1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const uint32_t idesc = idesc_bf16(kBM * kPair, mma_n(g.n0));
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#ifdef LP_GEMM_PROF
          if (n_mma++ == 0 && lane == 0) GEMM_PROF(4);  // first operands landed
#endif
          if (elect_one()) {
            const uint64_t a_desc = sdesc_sw128(smem_u32(sA + stage * C::kABytes));
            const uint64_t b_desc = sdesc_sw128(smem_u32(sB + stage * C::kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // +32 bytes per UMMA_K=16 slice inside the swizzle atom (>>4 => +2).
              const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
              if constexpr (kPair == 2) tc_mma_bf16_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, accum);
              else tc_mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, accum);
            }
            if constexpr (kPair == 2) tc_commit_pair(&empty[stage]);
            else tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if constexpr (kPair == 2) tc_commit_pair(&tfull[acc]);
          else tc_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
      if (lane == 0) GEMM_PROF(5);  // last MMA committed
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // Groups of 4 warps; each covers all 128 TMEM lanes (warp w may touch
    // lanes 32*(w%4)..+31) and takes every kEpiGroups-th 16-column chunk. The
    // fused QKV/RoPE epilogue (opt-in) runs on group 0 alone (its staging is 17 KB).
    const int q = warp % 4;                 // TMEM lane quarter this warp may touch
    const int row = q * 32 + lane;          // tile row == TMEM lane
    const int eg = (warp - 2) / 4;          // epilogue group
    const int et = threadIdx.x - 64 - eg * 128;  // 0..127 within the group
    const bool solo = args.mode == kEpiQkvRope;
    const int c_first = solo ? 0 : eg * 16, c_step = solo ? 16 : 16 * kEpiGroups;
    const bool idle = solo && eg == 1;
    __nv_bfloat16* const stage_g =
        eg == 0 ? epi_stage : reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(epi_stage) + 2 * kEpiStageBytes);
    const uint32_t tempty_leader = kPair == 2 ? mapa(smem_u32(&tempty[0]), 0) : 0;
    int acc = 0;
    uint32_t aphase = 0;
    int sbuf = 0;
    int it = first_it();
    Seg g;
#ifdef LP_GEMM_PROF
    int n_epi = 0;
#endif
    while (next_seg(it, g)) {
      const int s = g.s, m0 = g.m0, n0 = g.n0;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
#ifdef LP_GEMM_PROF
      if (et == 0 && eg == 0) {
        if (n_epi == 0) GEMM_PROF(6);  // first accumulator ready
        GEMM_PROF(8);                  // last accumulator ready (overwritten per unit)
      }
      ++n_epi;
#endif
      const int m = m0 + row;
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      float bias = 0.f;
      if (args.mode == kEpiBf16 && args.bias)
        bias = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.bias)[m]);
      const int ncols = min(tw, n_live - n0);  // live tokens of this tile
      const size_t ldm = static_cast<size_t>(args.M);
      float* const ws_unit = args.ws + static_cast<size_t>(s) * args.ws_stride * ldm + m;  // fp32 partial modes
      // Stream-K: record the tile's segment count once (its first segment),
      // for the reduction kernel, which sums slices 0..nseg-1 in order.
      if (sk && g.seg == 0 && et == 0 && eg == 0) {
        args.sk_tab[kSkTabHeader + g.tile] = g.nseg;
        if (g.tile == 0) {
          args.sk_tab[0] = tw;
          args.sk_tab[1] = sk_tiles_n;
          args.sk_tab[2] = kBM * kPair;
        }
      }
#ifdef LP_GEMM_PROF
      long long p_ld = 0, p_st = 0, p_t = clock64();
#endif
      // TMEM loads run one 16-column chunk ahead of the stores: the next
      // chunk's round trip overlaps this chunk's global writes.
      const int c_end = idle ? 0 : ncols;
      uint32_t nxt[16];
      if (c_first < c_end) tmem_ld16_issue(t_addr + c_first, nxt);
#pragma unroll 1
      for (int c = c_first; c < c_end; c += c_step) {  // uniform across the epilogue group
        float v[16];
        tmem_ld16_wait(nxt);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(nxt[j]);
        if (c + c_step < c_end) tmem_ld16_issue(t_addr + c + c_step, nxt);
#ifdef LP_GEMM_PROF
        { const long long now = clock64(); p_ld += now - p_t; p_t = now; }
#endif
        const int nbase = n0 + c;
        const int cnt = min(16, ncols - c);
        if (args.mode == kEpiF32Partial) {
          // 32 lanes x consecutive m: one full 128-byte line per token. One
          // warp per SM sub-partition runs this, so it is latency-bound:
          // every address is an independent offset from one base (no
          // dependent chains), and full chunks store unpredicated.
          float* dst = ws_unit + static_cast<size_t>(nbase) * ldm;
          if (cnt == 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[j * ldm] = v[j];
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < cnt) dst[j * ldm] = v[j];
          }
        } else if (args.mode == kEpiSiluMul) {
          // Even row = gate, odd row = up of feature m/2. Stage the 64-feature x
          // 16-token block in smem, then write 128-byte token rows with 16-byte
          // vector stores.
          // Lane pair (2f, 2f+1) holds gate / up of feature f for 16 tokens.
          // One shuffle per two tokens: the even lane finishes token j, the
          // odd lane token j+1, so every lane does useful work.
          __nv_bfloat16* stg = stage_g + sbuf * (16 * 64);
          const bool odd = lane & 1;
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float other = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[j + 1], 1);
            // Projections are rounded to bf16 before the activation (oracle storage point).
            const float g = __bfloat162float(__float2bfloat16_rn(odd ? other : v[j]));
            const float u = __bfloat162float(__float2bfloat16_rn(odd ? v[j + 1] : other));
            stg[(j + (odd ? 1 : 0)) * 64 + (row >> 1)] = __float2bfloat16_rn(silu(g) * u);
          }
          epi_bar(eg);
          const int tj = et >> 3, seg = et & 7;
          if (tj < cnt) {
            const uint4 val = *reinterpret_cast<const uint4*>(stg + tj * 64 + seg * 8);
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) +
                                 static_cast<size_t>(nbase + tj) * args.ldo + (m0 >> 1) + seg * 8;
            *reinterpret_cast<uint4*>(dst) = val;
          }
          sbuf ^= 1;
        } else if (args.mode == kEpiResidAdd) {
          // All 16 residual loads are issued before the first store: the
          // compiler cannot reorder a load above a possibly-aliasing store.
          float* dst = args.resid + static_cast<size_t>(nbase) * args.M + m;
          float r[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = j < cnt ? dst[static_cast<size_t>(j) * args.M] : 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < cnt) dst[static_cast<size_t>(j) * args.M] = r[j] + v[j];
        } else if (args.mode == kEpiQkvRope) {
          // This CTA's 128 rows are one head (head_dim 128): bias, then RoPE
          // for q/k heads (rotate-half pairs (i, i+64) live in warps q and
          // q^2: exchanged through smem), then bf16 out to q or the KV page.
          const QkvEpi& e = args.qkv;
          const int hd = m0 >> 7;
          const float b = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.bias)[m]);
          // Per-token metadata into registers before any store (see ResidAdd).
          int pos[16], slot[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            pos[j] = j < cnt ? e.positions[nbase + j] : 0;
            slot[j] = j < cnt ? e.slots[nbase + j] : 0;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += b;
          if (hd < e.nq + e.nkv) {  // uniform per CTA
            float* xs = reinterpret_cast<float*>(stage_g) + sbuf * (128 * 17);
#pragma unroll
            for (int j = 0; j < 16; ++j) xs[row * 17 + j] = v[j];
            epi_bar(eg);
            const int prow = row ^ 64;
            const float f = e.inv_freq[row & 63];
            const float sgn = row < 64 ? -1.f : 1.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float p = xs[prow * 17 + j];
              float sn, cs;
              sincosf(static_cast<float>(pos[j]) * f, &sn, &cs);
              v[j] = v[j] * cs + sgn * p * sn;
            }
            sbuf ^= 1;
          }
          if (hd < e.nq) {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(e.q_out) + static_cast<size_t>(nbase) * e.nq * 128 + m;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < cnt) dst[static_cast<size_t>(j) * e.nq * 128] = __float2bfloat16_rn(v[j]);
          } else {
            const bool is_v = hd >= e.nq + e.nkv;
            const int g = is_v ? hd - e.nq - e.nkv : hd - e.nq;
            const size_t page_elems = static_cast<size_t>(2) * e.nkv * e.page_size * 128;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j < cnt) {
                const int page = slot[j] / e.page_size, s_in = slot[j] % e.page_size;
                __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(e.kv_layer) + page * page_elems +
                                     ((static_cast<size_t>(is_v ? 1 : 0) * e.nkv + g) * e.page_size + s_in) * 128 + row;
                *dst = __float2bfloat16_rn(v[j]);
              }
            }
          }
        } else if (args.mode == kEpiBf16) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) +
                               static_cast<size_t>(nbase) * args.ldo + m;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < cnt) dst[static_cast<size_t>(j) * args.ldo] = __float2bfloat16_rn(v[j] + bias);
        } else {  // kEpiF32
          float* dst = reinterpret_cast<float*>(args.out) + static_cast<size_t>(nbase) * args.ldo + m;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < cnt) dst[static_cast<size_t>(j) * args.ldo] = v[j];
        }
#ifdef LP_GEMM_PROF
        { const long long now = clock64(); p_st += now - p_t; p_t = now; }
#endif
      }
#ifdef LP_GEMM_PROF
      if (et == 0 && eg == 0 && args.M == g_gemm_prof_sel[0] && args.K == g_gemm_prof_sel[1] && blockIdx.x < kProfCtas) {
        g_gemm_prof[blockIdx.x][10] = p_ld;
        g_gemm_prof[blockIdx.x][11] = p_st;
      }
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair == 2) mbar_arrive_remote(tempty_leader + acc * 8);
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
#ifdef LP_GEMM_PROF
    if (et == 0 && eg == 0) {
      GEMM_PROF(7);  // epilogue done
      if (args.M == g_gemm_prof_sel[0] && args.K == g_gemm_prof_sel[1] && blockIdx.x < kProfCtas)
        g_gemm_prof[blockIdx.x][9] = n_epi;
    }
#endif
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (kPair == 2) cluster_sync();  // the peer may still signal our barriers
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair == 2) tmem_dealloc_pair<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    }
    fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

template <int BN, int kPair>
void launch_bn(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
               cudaStream_t stream, int max_ctas) {
  using C = Cfg<BN, kPair>;
  auto* kern = gemm_bf16_tn_kernel<BN, kPair>;
  smem_attr_once(reinterpret_cast<const void*>(kern), C::kSmem);
  // Stream-K from the host (splits < 0): one CTA (pair) per SM (pair).
  const int units = a.splits < 0 ? (1 << 30)
                                 : a.splits * (a.M / (kBM * kPair)) * std::max((a.N + BN - 1) / BN, a.n_tiles_cap);
  int grid = num_sms() / kPair;
  if (max_ctas > 0 && max_ctas / kPair < grid) grid = max_ctas / kPair;
  if (units < grid) grid = units;
  grid *= kPair;
  if constexpr (kPair == 1) {
    launch_k(kern, dim3(grid), dim3(kThreads), C::kSmem, stream, tmA, tmB, a);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, tmA, tmB, a);
  }
}

}  // namespace

#ifdef LP_GEMM_PROF
extern "C" int lp_debug_gemm_prof(unsigned long long* out, size_t n, int M, int K) {
  const int sel[2] = {M, K};
  static unsigned long long zero[kProfCtas][kProfEv];
  const size_t bytes = std::min(n * sizeof(unsigned long long), sizeof(g_gemm_prof));
  if (out && cudaMemcpyFromSymbol(out, g_gemm_prof, bytes) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(g_gemm_prof, zero, sizeof(zero)) != cudaSuccess) return -1;
  return cudaMemcpyToSymbol(g_gemm_prof_sel, sel, sizeof(sel)) == cudaSuccess ? 0 : -1;
}
#endif

int num_sms() {
  // Per device: a process may drive several GPUs (one instance each).
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev & 63];
  int n = slot.load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    slot.store(n, std::memory_order_relaxed);
  }
  return n;
}

CUtensorMap make_tmap_bf16(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  }
  return m;
}

int gemm_b_box_rows(int bn, int pair) { return bn / pair; }

CUtensorMap make_tmap_3d_bf16(const void* ptr, const uint64_t dims[3], const uint64_t strides_bytes[2],
                              const uint32_t box[3]) {
  CUtensorMap m;
  const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t s[2] = {strides_bytes[0], strides_bytes[1]};
  const cuuint32_t b[3] = {box[0], box[1], box[2]};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), d, s, b,
                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled (3d) failed: " + std::to_string(static_cast<int>(r)));
  }
  return m;
}

void gemm_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, int bn,
                 cudaStream_t stream, int max_ctas, int pair) {
  const bool sk = a.splits < 0;
  if (sk && (a.mode != kEpiF32Partial || !a.sk_tab || !a.ws))
    throw std::runtime_error("gemm_launch: stream-K needs fp32 partial output, a workspace and a segment table");
  if (a.M % (kBM * pair) != 0 || a.K % kBK != 0 || a.N < 1 || a.splits == 0) {
    throw std::runtime_error("gemm_launch: unsupported shape M=" + std::to_string(a.M) +
                             " K=" + std::to_string(a.K) + " N=" + std::to_string(a.N) +
                             " pair=" + std::to_string(pair));
  }
  if (a.mode == kEpiSiluMul && (a.ldo % 8 != 0)) throw std::runtime_error("gemm_launch: SiLU ldo % 8");
  if (pair == 2) {
    switch (bn) {
      case 32: launch_bn<32, 2>(tmA, tmB, a, stream, max_ctas); return;
      case 64: launch_bn<64, 2>(tmA, tmB, a, stream, max_ctas); return;
      case 128: launch_bn<128, 2>(tmA, tmB, a, stream, max_ctas); return;
      case 256: launch_bn<256, 2>(tmA, tmB, a, stream, max_ctas); return;
      default: throw std::runtime_error("gemm_launch: bad paired bn " + std::to_string(bn));
    }
  }
  switch (bn) {
    case 16: launch_bn<16, 1>(tmA, tmB, a, stream, max_ctas); break;
    case 32: launch_bn<32, 1>(tmA, tmB, a, stream, max_ctas); break;
    case 64: launch_bn<64, 1>(tmA, tmB, a, stream, max_ctas); break;
    case 128: launch_bn<128, 1>(tmA, tmB, a, stream, max_ctas); break;
    case 256: launch_bn<256, 1>(tmA, tmB, a, stream, max_ctas); break;
    default: throw std::runtime_error("gemm_launch: bad bn " + std::to_string(bn));
  }
}

}  // namespace lp

KTL_EXPORT(gemm)
