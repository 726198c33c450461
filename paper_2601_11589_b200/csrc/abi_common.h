// Error plumbing for the C ABI: no C++ exception ever crosses the boundary.
// Every entry point runs its body under lp_guard, which maps exceptions to
// negative status codes and records the message for lp_last_error().
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/laps_prefill.h"

namespace lp {

struct ShapeMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {  // call out of order / expired ticket
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

inline void lp_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename F>
int lp_guard(F&& f) {
  try {
    f();
    return LP_OK;
  } catch (const ShapeMismatch& e) {
    set_last_error(e.what());
    return LP_ERR_SHAPE;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return LP_ERR_CONFIG;
  } catch (const OutOfMemory& e) {
    set_last_error(e.what());
    return LP_ERR_OOM;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return LP_ERR_CUDA;
  } catch (const StateError& e) {
    set_last_error(e.what());
    return LP_ERR_STATE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return LP_ERR_INTERNAL;
  }
}

}  // namespace lp
