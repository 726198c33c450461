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

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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
