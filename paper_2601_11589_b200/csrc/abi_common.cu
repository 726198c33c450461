#include <cuda_bf16.h>

#include <cstring>
#include <mutex>
#include <string>

#include "abi_common.h"
#include "synth.h"

namespace lp {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace lp

extern "C" {

const char* lp_last_error(void) { return lp::g_last_error.c_str(); }

const char* lp_version(void) { return "laps-b200 0.1 (sm_100a)"; }

int32_t lp_synth_token(uint64_t seed, int64_t session_id, int64_t position, int32_t vocab) {
  return lp::synth_token(seed, session_id, position, vocab);
}

// Test hook: bf16 bits of weight element `index` of tensor `tensor_id`, from
// the same generator + RNE conversion the device init kernel uses (host side).
uint16_t lpk_synth_weight_bits(uint64_t seed, uint64_t tensor_id, uint64_t index, float scale) {
  const __nv_bfloat16 b = __float2bfloat16_rn(lp::synth_weight_f32(seed, tensor_id, index, scale));
  uint16_t bits;
  memcpy(&bits, &b, 2);
  return bits;
}

}  // extern "C"
