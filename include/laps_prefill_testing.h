/*
 * laps_prefill_testing.h — kernel-level test hooks of liblaps_prefill.so.
 *
 * NOT part of the drop-in boundary (that is laps_prefill.h). These entry
 * points let the parity tests and the measurement scripts drive single
 * sm_100a kernels on raw device pointers or time one projection inside an
 * instance. Same conventions as laps_prefill.h: int status, LP_ERR_* codes,
 * lp_last_error() for the text, no exceptions across the boundary.
 */
#ifndef LAPS_PREFILL_TESTING_H_
#define LAPS_PREFILL_TESTING_H_

#include <stdint.h>

#include "laps_prefill.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Epilogue modes of lpk_gemm (csrc/gemm_sm100.cuh kEpi*). */
#define LPK_EPI_BF16 0        /* out_bf16[n*ldo + m] = acc (+ bias[m]) */
#define LPK_EPI_F32_PARTIAL 1 /* fp32 split-K partials ws[(split*N + n)*M + m] */
#define LPK_EPI_SILU_MUL 2    /* row-interleaved gate/up -> bf16 SiLU(gate)*up */
#define LPK_EPI_F32 3         /* out_f32[n*ldo + m] = acc */

/* One tcgen05 GEMM launch: out[N, M] = X[N, K] . W[M, K]^T on `stream`
 * (cudaStream_t), device pointers only. bn = token tile (16..256), pair = 1
 * or 2 (cta_group::2), n_dev = device int holding the live token count. */
int lpk_gemm(const void* W, const void* X, void* out, float* ws, const void* bias, int M, int N, int K,
             int splits, int mode, int bn, int ldo, const int* n_dev, void* stream, int pair);

/* Stream-K launch of the same GEMM (fp32 partial output): the grid's CTAs
 * (pairs), at most max_ctas CTAs (0 = one per SM), split the (tile, 64-deep
 * K block) steps evenly, so a tile is cut into 1..n segments; segment j of a
 * tile lands in ws slice j (ws holds n slices of N x M) and the segment
 * counts in seg_table: [0] token-tile width, [1] token tiles, [2] weight rows
 * per tile, [4 + m_tile * tiles + n_tile] segments. */
int lpk_gemm_stream_k(const void* W, const void* X, float* ws, int M, int N, int K, int bn, int pair,
                      const int* n_dev, int* seg_table, int max_ctas, void* stream);

/* Time one projection of layer `layer` inside an instance (which: 0 QKV,
 * 1 O, 2 gate/up + SiLU, 3 down) at capacity t_cap with n_live live tokens:
 * *avg_ms = mean CUDA-event time over `iters` back-to-back launches. */
int lpk_time_gemm(lp_instance* inst, int32_t layer, int32_t which, int32_t t_cap, int32_t n_live,
                  int32_t iters, double* avg_ms);

/* Attention schedule of the last submit: *pieces work pieces (persistent
 * tcgen05 grid) or work items, *merges units split across CTAs (merged by
 * their last piece), *ctas CTAs with work. */
int lpk_last_attention_schedule(lp_instance* inst, int32_t* pieces, int32_t* merges, int32_t* ctas);

/* The GEMM launch planner on the host alone (no GPU): the capacity plan of a
 * projection [M out, K in] at t_cap tokens (token tile bn, CTA pair) and the
 * per-batch (token tiles, split-K) choice for n_live live tokens on `sms` SMs
 * (allow_split = 0: fused epilogues, one K slice). */
int lpk_plan_gemm(int32_t M, int32_t K, int32_t t_cap, int32_t n_live, int32_t sms, int32_t allow_split,
                  int32_t* bn, int32_t* pair, int32_t* n_tiles, int32_t* splits);

/* The persistent attention's planner on the host alone (no GPU): blocks of
 * `needs[i]` pages (heaviest first) x nkv kv heads onto ncta lists. out
 * (capacity `cap` pieces) receives per piece {cta, block, kv head, first page,
 * end page, merge entry or -1}; *lpt_span = -1 when the split lists were
 * chosen, else the whole-unit makespan; *list_cap = the McNaughton capacity
 * (steps). */
int lpk_plan_attention(const int32_t* needs, int32_t n_blocks, int32_t nkv, int32_t ncta, int32_t* out,
                       int32_t cap, int32_t* n_pieces, int32_t* n_merges, double* list_cap, double* lpt_span);

/* bf16 bits of weight element `index` of tensor `tensor_id` from the device
 * initialiser's generator (host side; the oracle must reproduce them). */
uint16_t lpk_synth_weight_bits(uint64_t seed, uint64_t tensor_id, uint64_t index, float scale);

#ifdef __cplusplus
}
#endif

#endif /* LAPS_PREFILL_TESTING_H_ */
