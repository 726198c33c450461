// Kernel launch with Programmatic Dependent Launch (PDL).
//
// Every kernel of the forward is launched with the programmatic stream
// serialization attribute (captured into the per-shape CUDA graphs as
// programmatic edges). Kernels call pdl_trigger() early so the next kernel's
// CTAs can become resident and run their prologue (barrier init, TMEM alloc,
// tensor-map prefetch and — for the GEMMs — the first weight tiles, which do
// not depend on the previous kernel) while this one drains; everything that
// reads a predecessor's output or writes shared buffers sits after
// pdl_wait(), which returns once all predecessor grids completed and flushed.
// Set LP_PDL=0 in the environment to launch without the attribute.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

namespace lp {

// Diagnostic build only (-DLP_KTL, scripts/kernel_timeline.py): block 0 /
// thread 0 of every forward kernel stamps %globaltimer at entry, after its
// PDL wait and at its exit into a device log (each translation unit holds
// the log's address in its own constant, set through lp_ktl_set_<unit>).
// Record: {kind << 32 | meta, entry, start, end}. Compiled out of the
// product library.
#ifdef LP_KTL
static __constant__ unsigned long long* c_ktl_log;  // [0] = record count, records of 4 from [4]
__device__ __forceinline__ unsigned long long ktl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool ktl_me() {
  return blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && c_ktl_log != nullptr;
}
// One slot per translation unit (no shared memory: some kernels use all of
// it). Only the running kernel's block 0 writes it from pdl_wait; the next
// kernel's wait returns after this one completed, so the slot holds this
// kernel's stamp at its exit (a stamp older than the entry = no wait seen).
static __device__ unsigned long long g_ktl_start;
__device__ __forceinline__ unsigned long long& ktl_start_slot() { return g_ktl_start; }
struct KtlScope {
  int kind, meta;
  unsigned long long t0 = 0;
  __device__ KtlScope(int k, int m) : kind(k), meta(m) {
    if (ktl_me()) t0 = ktl_now();
  }
  __device__ ~KtlScope() {
    if (ktl_me()) {
      const unsigned long long i = atomicAdd(c_ktl_log, 1ull);
      if (i < 16383) {
        unsigned long long* r = c_ktl_log + 4 + 4 * i;
        r[0] = (static_cast<unsigned long long>(kind) << 32) | static_cast<unsigned int>(meta);
        r[1] = t0;
        r[2] = ktl_start_slot();
        r[3] = ktl_now();
      }
    }
  }
};
#define KTL_SCOPE(kind, meta) ::lp::KtlScope ktl_scope_((kind), (meta))
#define KTL_EXPORT(unit)                                                          \
  extern "C" int lp_ktl_set_##unit(void* p) {                                     \
    return cudaMemcpyToSymbol(lp::c_ktl_log, &p, sizeof(p)) == cudaSuccess ? 0 : -1; \
  }
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (ktl_me()) ktl_start_slot() = ktl_now();
}
#else
#define KTL_SCOPE(kind, meta) (void)0
#define KTL_EXPORT(unit)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
// Kernel kinds of the log.
enum KtlKind : int { kKtlGemm = 1, kKtlQkvPost = 2, kKtlResidNorm = 3, kKtlEmbed = 4, kKtlAttnWarp = 5,
                     kKtlAttnCombine = 6, kKtlAttnTc = 7, kKtlAttnTcp = 8, kKtlGather = 9, kKtlArgmax = 10 };
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Timing experiments only (results are wrong): LP_DEBUG_EMPTY lists kernel
// classes ("norm", "qkv", "attn") whose launches are replaced by an empty PDL
// kernel of the same grid, to split a forward's time into kernel work and
// kernel-boundary cost.
inline bool debug_empty(const char* cls) {
  const char* e = std::getenv("LP_DEBUG_EMPTY");
  return e && std::strstr(e, cls) != nullptr;
}
void launch_empty(dim3 grid, dim3 block, cudaStream_t st);

// Raise a kernel's dynamic shared-memory limit on the CURRENT device, once
// per (kernel, device). The attribute lives in the device's context, so a
// process driving several GPUs (one instance per device, possibly from
// different host threads) must set it on every device it launches on.
inline void smem_attr_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kernel, dev})) return;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("cudaFuncSetAttribute(max dynamic smem): ") + cudaGetErrorString(e));
  done.insert({kernel, dev});
}

}  // namespace lp
