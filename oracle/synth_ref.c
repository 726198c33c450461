/*
 * TEST INFRASTRUCTURE — CPU restatement of the deterministic input / weight
 * generators (the product's copy is paper_2601_11589_b200/csrc/synth.h).
 * Integer arithmetic plus one IEEE fp32 multiply and a round-to-nearest-even
 * bf16 conversion, so results are bit-identical to the GPU.
 *
 * The reference has no model and no token content:
 * these generators define the synthetic inputs the parity tests share.
 *
 * Build: see oracle/Makefile (`make -C oracle synth`).
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) { return sm64(sm64(sm64(a) ^ b) ^ c); }

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

int32_t oracle_token(uint64_t seed, int64_t session, int64_t pos, int32_t vocab) {
  return (int32_t)(mix3(seed, (uint64_t)session, (uint64_t)pos) % (uint64_t)vocab);
}

void oracle_tokens(uint64_t seed, int64_t session, int64_t pos0, int64_t n, int32_t vocab, int32_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_token(seed, session, pos0 + i, vocab);
}

/* out[i] = bf16(float(q) * scale), q = (mix3(seed, tid, i) >> 40) - 2^23.
 * interleave != 0: `out` is the [2*rows, cols] row interleave of tensors tid
 * (even rows) and tid+1 (odd rows). Rows [row0, row0+nrows) only. */
void oracle_weights_bf16(uint16_t* out, int64_t row0, int64_t nrows, int64_t cols, uint64_t seed,
                         uint64_t tid, float scale, int interleave) {
  for (int64_t r = row0; r < row0 + nrows; ++r) {
    uint64_t t = tid;
    int64_t lr = r;
    if (interleave) {
      t = tid + (uint64_t)(r & 1);
      lr = r >> 1;
    }
    uint16_t* dst = out + (r - row0) * cols;
    for (int64_t c = 0; c < cols; ++c) {
      const uint64_t h = mix3(seed, t, (uint64_t)(lr * cols + c));
      const int32_t q = (int32_t)(h >> 40) - (1 << 23);
      dst[c] = f32_to_bf16_rne((float)q * scale);
    }
  }
}
