// Microbenchmark: per-SM throughput of MUFU.EX2, FFMA, FFMA2 and the degree-5
// polynomial exp2 on this GPU (ops per clock per SM, from CUDA events and the
// SM clock read by clock64 inside the kernel).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/pipe_rates scripts/repro/pipe_rates.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int kMode>
__global__ void bench(float* out, long long* clk, float a, float b) {
  float v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) v[i] = threadIdx.x * 1e-3f + i;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if constexpr (kMode == 0) v[i] = ex2(v[i] * -1e-3f);                  // 1 MUFU + 1 FMUL
      else if constexpr (kMode == 1) v[i] = fmaf(v[i], a, b);                // 1 FFMA
      else if constexpr (kMode == 3) {                                       // 1 F2FP bf16x2 pack per 2 chains
        if (i % 2 == 0) {
          uint32_t r;
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i + 1]), "f"(v[i]));
          v[i] = __uint_as_float(r) ;
          v[i + 1] = __uint_as_float(r ^ 0x1u);
        }
      } else if constexpr (kMode == 4) {                                     // integer round-half-up pack
        if (i % 2 == 0) {
          const uint32_t lo = __float_as_uint(v[i]) + 0x8000u, hi = __float_as_uint(v[i + 1]) + 0x8000u;
          const uint32_t r = __byte_perm(lo, hi, 0x7632);
          v[i] = __uint_as_float(r);
          v[i + 1] = __uint_as_float(r ^ 0x1u);
        }
      }
      else if constexpr (kMode == 2) {                                       // 1 FFMA2 per 2 chains
        if (i % 2 == 0) {
          float2 r;
          asm("{.reg .b64 x, y, z, d;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %4};\n mov.b64 z, {%5, %5};\n"
              " fma.rn.f32x2 d, x, y, z;\n mov.b64 {%0, %1}, d;}"
              : "=f"(r.x), "=f"(r.y) : "f"(v[i]), "f"(v[i + 1]), "f"(a), "f"(b));
          v[i] = r.x;
          v[i + 1] = r.y;
        }
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int blocks_per_sm, int sms, double ops_per_thread_iter) {
  const int blocks = blocks_per_sm * sms, threads = 256;
  float* out;
  long long* clk;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&clk, sizeof(long long) * blocks);
  bench<kMode><<<blocks, threads>>>(out, clk, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  bench<kMode><<<blocks, threads>>>(out, clk, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  // blocks_per_sm resident blocks share one SM for the whole run
  const double ops_per_sm = ops_per_thread_iter * kIters * threads * blocks_per_sm;
  std::printf("%-28s %6.1f ops/clk/SM  (%d blocks/SM x 256 threads, %lld cycles)\n", name, ops_per_sm / mx,
              blocks_per_sm, mx);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int b : {2, 4, 8}) {
    run<0>("MUFU.EX2 (+FMUL)", b, sms, kChains);
    run<1>("FFMA", b, sms, kChains);
    run<2>("FFMA2 (lane ops)", b, sms, kChains);
    run<3>("F2FP bf16x2 (values)", b, sms, kChains);
    run<4>("int RN pack (values)", b, sms, kChains);
  }
  return 0;
}
