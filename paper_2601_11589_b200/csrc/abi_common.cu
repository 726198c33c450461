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

}  // extern "C"
