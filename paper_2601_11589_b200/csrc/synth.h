// Counter-based deterministic generators shared by the CUDA path and the
// CPU oracle (oracle/forward_oracle.py restates them bit-for-bit):
//   * token ids  : splitmix64(seed, session, position) mod vocab
//   * weights    : splitmix64(seed, tensor_id, index) -> 24-bit integer ->
//                  exact fp32 scaling -> bf16 (round to nearest even)
// All arithmetic is integer or a single IEEE fp32 multiply, so CPU and GPU
// produce identical bits.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define LP_HD __host__ __device__ __forceinline__
#else
#define LP_HD inline
#endif

namespace lp {

LP_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

LP_HD uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) {
  return splitmix64(splitmix64(splitmix64(a) ^ b) ^ c);
}

LP_HD int32_t synth_token(uint64_t seed, int64_t session, int64_t pos, int32_t vocab) {
  return static_cast<int32_t>(mix3(seed, static_cast<uint64_t>(session), static_cast<uint64_t>(pos)) %
                              static_cast<uint64_t>(vocab));
}

// Uniform value in [-scale*2^23, scale*2^23) with 2^24 levels; returns the
// fp32 product (exact integer times power-of-two-free scale: one rounding).
LP_HD float synth_weight_f32(uint64_t seed, uint64_t tensor_id, uint64_t index, float scale) {
  const uint64_t h = mix3(seed, tensor_id, index);
  const int32_t q = static_cast<int32_t>(h >> 40) - (1 << 23);  // [-2^23, 2^23)
  return static_cast<float>(q) * scale;
}

}  // namespace lp
