// tcgen05 GEMM — see gemm_sm100.cuh for the orientation and roles.
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm_sm100.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace lp {

namespace {

constexpr int kBM = 128;            // weight rows per tile (MMA M)
constexpr int kBK = 64;             // K per stage: one 128-byte swizzle row of bf16
constexpr int kThreads = 192;       // warp0 TMA, warp1 MMA, warps2-5 epilogue
constexpr int kSmemBudget = 196 * 1024;
constexpr int kEpiStageBytes = 16 * 64 * 2;  // [16 tokens][64 features] bf16

template <int BN>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;   // 16 KiB
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmem = 1024 /*align*/ + kStages * kStageBytes + kBarBytes + 2 * kEpiStageBytes;
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  using C = Cfg<BN>;
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
  pdl_trigger();

  // n_dev is written by the pre-graph H2D copy, never by a kernel: safe before pdl_wait.
  const int n_live = args.n_dev ? min(*args.n_dev, args.N) : args.N;
  const int m_tiles = args.M / kBM;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_kb = args.K / kBK;
  const int splits = args.splits;
  const int units = splits * m_tiles * n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int w, int& s, int& m0, int& n0, int& kb0, int& kb1) {
    const int n = w % n_tiles;
    const int rest = w / n_tiles;
    const int m = rest % m_tiles;
    s = rest / m_tiles;
    m0 = m * kBM;
    n0 = n * BN;
    const int base = num_kb / splits, rem = num_kb % splits;
    kb0 = s * base + min(s, rem);
    kb1 = kb0 + base + (s < rem ? 1 : 0);
  };

  if (warp == 0) {
    // ----------------------------------------------------------- TMA producer
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once
      const uint64_t pol_x = policy_evict_last();   // activations are re-read per m tile
      // Weight tiles do not depend on the previous kernel: fill the pipeline
      // with them before waiting on it (PDL), then add the activation tiles.
      int pre = 0;
      int pre_w = -1, pre_kb0 = 0, pre_m0 = 0, pre_n0 = 0;
      for (int w = blockIdx.x; w < units; w += gridDim.x) {
        int s, m0, n0, kb0, kb1;
        decode(w, s, m0, n0, kb0, kb1);
        if (n0 >= n_live) continue;
        pre_w = w; pre_kb0 = kb0; pre_m0 = m0; pre_n0 = n0;
        pre = min(kb1 - kb0, C::kStages);
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], C::kStageBytes);
          tma_load_2d(sA + i * C::kABytes, &tmA, &full[i], (kb0 + i) * kBK, m0, pol_w);
        }
        break;
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sB + i * C::kBBytes, &tmB, &full[i], (pre_kb0 + i) * kBK, pre_n0, pol_x);
      (void)pre_m0;
      int stage = pre % C::kStages;
      uint32_t phase = pre == C::kStages ? 1u : 0u;
      for (int w = (pre_w >= 0 ? pre_w : units); w < units; w += gridDim.x) {
        int s, m0, n0, kb0, kb1;
        decode(w, s, m0, n0, kb0, kb1);
        if (n0 >= n_live) continue;
        for (int kb = (w == pre_w ? kb0 + pre : kb0); kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * kBK, m0, pol_w);
          tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBK, n0, pol_x);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(kBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int w = blockIdx.x; w < units; w += gridDim.x) {
      int s, m0, n0, kb0, kb1;
      decode(w, s, m0, n0, kb0, kb1);
      if (n0 >= n_live) continue;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t a_desc = sdesc_sw128(smem_u32(sA + stage * C::kABytes));
          const uint64_t b_desc = sdesc_sw128(smem_u32(sB + stage * C::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // +32 bytes per UMMA_K=16 slice inside the swizzle atom (>>4 => +2).
            tc_mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc,
                        (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) tc_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    const int q = warp % 4;          // TMEM lane quarter this warp may touch
    const int row = q * 32 + lane;   // tile row == TMEM lane
    const int et = threadIdx.x - 64; // 0..127 within the epilogue group
    int acc = 0;
    uint32_t aphase = 0;
    int sbuf = 0;
    for (int w = blockIdx.x; w < units; w += gridDim.x) {
      int s, m0, n0, kb0, kb1;
      decode(w, s, m0, n0, kb0, kb1);
      if (n0 >= n_live) continue;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int m = m0 + row;
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      float bias = 0.f;
      if (args.mode == kEpiBf16 && args.bias)
        bias = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.bias)[m]);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (n0 + c >= n_live) break;  // uniform across the epilogue group
        float v[16];
        tmem_ld16(t_addr + c, v);
        const int nbase = n0 + c;
        const int cnt = min(16, n_live - nbase);
        if (args.mode == kEpiF32Partial) {
          // 32 lanes x consecutive m: one full 128-byte line per token.
          float* dst = args.ws + (static_cast<size_t>(s) * args.ws_stride + nbase) * args.M + m;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < cnt) dst[static_cast<size_t>(j) * args.M] = v[j];
        } else if (args.mode == kEpiSiluMul) {
          // Even row = gate, odd row = up of feature m/2. Stage the 64-feature x
          // 16-token block in smem, then write 128-byte token rows with 16-byte
          // vector stores.
          __nv_bfloat16* stg = epi_stage + sbuf * (16 * 64);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float u = __shfl_xor_sync(0xffffffffu, v[j], 1);
            if ((lane & 1) == 0) {
              // Projections are rounded to bf16 before the activation (oracle storage point).
              const float g = __bfloat162float(__float2bfloat16_rn(v[j]));
              const float uu = __bfloat162float(__float2bfloat16_rn(u));
              stg[j * 64 + (row >> 1)] = __float2bfloat16_rn(silu(g) * uu);
            }
          }
          epi_bar();
          const int tj = et >> 3, seg = et & 7;
          if (tj < cnt) {
            const uint4 val = *reinterpret_cast<const uint4*>(stg + tj * 64 + seg * 8);
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) +
                                 static_cast<size_t>(nbase + tj) * args.ldo + (m0 >> 1) + seg * 8;
            *reinterpret_cast<uint4*>(dst) = val;
          }
          sbuf ^= 1;
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
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

template <int BN>
void launch_bn(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
               cudaStream_t stream, int max_ctas) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::kSmem);
    attr_set = true;
  }
  const int units = a.splits * (a.M / kBM) * ((a.N + BN - 1) / BN);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (units < grid) grid = units;
  launch_k(gemm_bf16_tn_kernel<BN>, dim3(grid), dim3(kThreads), C::kSmem, stream, tmA, tmB, a);
}

}  // namespace

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
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

void gemm_launch(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, int bn,
                 cudaStream_t stream, int max_ctas) {
  if (a.M % kBM != 0 || a.K % kBK != 0 || a.N < 1 || a.splits < 1) {
    throw std::runtime_error("gemm_launch: unsupported shape M=" + std::to_string(a.M) +
                             " K=" + std::to_string(a.K) + " N=" + std::to_string(a.N));
  }
  if (a.mode == kEpiSiluMul && (a.ldo % 8 != 0)) throw std::runtime_error("gemm_launch: SiLU ldo % 8");
  switch (bn) {
    case 16: launch_bn<16>(tmA, tmB, a, stream, max_ctas); break;
    case 32: launch_bn<32>(tmA, tmB, a, stream, max_ctas); break;
    case 64: launch_bn<64>(tmA, tmB, a, stream, max_ctas); break;
    case 128: launch_bn<128>(tmA, tmB, a, stream, max_ctas); break;
    case 256: launch_bn<256>(tmA, tmB, a, stream, max_ctas); break;
    default: throw std::runtime_error("gemm_launch: bad bn " + std::to_string(bn));
  }
}

}  // namespace lp
