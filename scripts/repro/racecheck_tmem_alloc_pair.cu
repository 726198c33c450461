// Minimal racecheck repro for the hazards compute-sanitizer reports on the
// CTA-pair GEMM (profiles/r02_sanitizer.txt): a cluster of 2 CTAs, warp 1 of
// each allocates TMEM with tcgen05.alloc.cta_group::2 (the hardware writes the
// allocated address into the shared-memory slot of BOTH CTAs), then the same
// fence / __syncthreads / barrier.cluster / fence sequence as gemm_sm100.cu,
// then every thread reads the slot. Variant 1 (argv[1] == "1") adds nothing
// else; variant 0 replaces the pair allocation with cta_group::1 (the CTA's
// own warp writes its own slot). racecheck flags variant 1 only: its write is
// unattributed (no thread performed it), so the tool cannot order it against
// the reads that the cluster barrier does order.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/repro_tmem scripts/repro/racecheck_tmem_alloc_pair.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kPair>
__global__ void __cluster_dims__(2, 1, 1) alloc_kernel(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 1) {
    if constexpr (kPair == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = slot;  // <- the read racecheck pairs with the unattributed write
  out[blockIdx.x * blockDim.x + threadIdx.x] = taddr;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    if constexpr (kPair == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(taddr));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(taddr));
  }
}

int main(int argc, char** argv) {
  const int pair = argc > 1 ? std::atoi(argv[1]) : 1;
  uint32_t* out = nullptr;
  cudaMalloc(&out, 2 * 128 * sizeof(uint32_t));
  if (pair) alloc_kernel<2><<<2, 128>>>(out);
  else alloc_kernel<1><<<2, 128>>>(out);
  const cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[256];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("variant %s: %s, CTA0 slot %u, CTA1 slot %u\n", pair ? "cta_group::2" : "cta_group::1",
              cudaGetErrorString(e), h[0], h[128]);
  cudaFree(out);
  return e == cudaSuccess ? 0 : 1;
}
