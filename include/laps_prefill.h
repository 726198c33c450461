/*
 * laps_prefill.h — C ABI of the B200-native LAPS prefill instance.
 *
 * This is the drop-in boundary for the reference's forward stand-in. In the
 * reference (prefillsim, /root/reference/proj) a dispatched batch's "forward"
 * is one closed-form call:
 *
 *   double batch_service_time(const BatchShape&, std::span<const MemberShape>,
 *                             const CostParams&, const ExecOverheads&);
 *       include/prefillsim/cost_model.hpp:117-119, src/cost_model.cpp:128-148
 *   double packed_service_time(std::span<const MemberShape>, ...);
 *       include/prefillsim/cost_model.hpp:124-125, src/cost_model.cpp:150-158
 *
 * called from exactly three engine sites: sim.cpp:254 (short/AWD batch),
 * sim.cpp:283 (long-prefill chunk), sim.cpp:357 (FCFS packed batch).
 * lp_submit() replaces those calls with a real Qwen2-style prefill forward
 * over a paged KV cache on one B200; lp_wait() returns the measured service
 * time that the reference computed analytically.
 *
 * Conventions
 *  - Every function returns int status: LP_OK (0) or a negative LP_ERR_*.
 *    LP_ERR_SHAPE mirrors prefillsim::ShapeMismatch (cost_model.hpp:78-80),
 *    LP_ERR_CONFIG mirrors prefillsim::ConfigError (cost_model.hpp:17-19).
 *    No C++ exception crosses this boundary; lp_last_error() has the text.
 *  - The caller owns every host array; the instance owns all device memory.
 *  - One instance == one GPU == one reference `Inst` (sim.cpp:95-112). Calls
 *    on one instance must be serialized; different instances may be driven
 *    from different host threads.
 *  - Plain pointers and sizes only; no framework types.
 */
#ifndef LAPS_PREFILL_H_
#define LAPS_PREFILL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_OK 0
#define LP_ERR_SHAPE (-1)    /* prefillsim::ShapeMismatch */
#define LP_ERR_CONFIG (-2)   /* prefillsim::ConfigError */
#define LP_ERR_OOM (-3)      /* KV page pool or HBM exhausted */
#define LP_ERR_CUDA (-4)     /* CUDA runtime failure */
#define LP_ERR_STATE (-5)    /* call out of order (e.g. wait without submit) */
#define LP_ERR_INTERNAL (-9)

/* Shape kinds: prefillsim::ShapeKind (cost_model.hpp:58) plus the unpadded
 * packed batch of the FCFS baseline (packed_service_time). */
#define LP_KIND_GRAPH 0
#define LP_KIND_STANDARD 1
#define LP_KIND_PACKED 2

typedef struct lp_instance lp_instance;

/* Qwen2-style decoder shape (random-init; the reference has no model). */
typedef struct lp_model_desc {
  int32_t hidden;        /* h */
  int32_t intermediate;  /* i */
  int32_t layers;
  int32_t n_q_heads;
  int32_t n_kv_heads;
  int32_t head_dim;      /* must be 64 or 128 */
  int32_t vocab;
  float rope_theta;
  float rms_eps;
  float init_std;        /* weights ~ U(-a, a) with std init_std */
  uint64_t weight_seed;
} lp_model_desc;

typedef struct lp_instance_desc {
  int32_t device;
  int32_t page_size;     /* tokens per KV page: 0 (default) or 64 — the attention key tile */
  int64_t kv_pages;      /* pool size in pages; 0 = size from free HBM */
  int64_t max_tokens;    /* activation arena capacity (tokens per forward) */
  int32_t max_members;   /* max requests per forward */
  int32_t use_graphs;    /* capture per-(l_pad, depth) CUDA graphs */
} lp_instance_desc;

/* prefillsim::BatchShape (cost_model.hpp:60-64) + packed kind. */
typedef struct lp_shape {
  int64_t l_pad;
  int32_t depth;
  int32_t kind;
} lp_shape;

/* prefillsim::MemberShape (cost_model.hpp:112) widened with identity: a
 * real forward needs to know whose KV it extends. Tokens [history,
 * history + new_tokens) of session `session_id` are computed; positions
 * [0, history) must already be resident (see lp_session_*). */
typedef struct lp_member {
  int64_t req_id;
  int64_t session_id;
  int64_t new_tokens;   /* L (or chunk length) */
  int64_t history;      /* H (+ preceding chunk tokens for long chunks) */
  int32_t want_logits;  /* produce first-token output for this member; when no
                           member of a forward sets it (an intermediate chunk
                           of a long prompt, a history fill) the LM head is
                           skipped and its first tokens read back as -1 */
  int32_t reserved;
} lp_member;

/* ---- instance lifecycle ---- */
int lp_instance_create(const lp_model_desc* model, const lp_instance_desc* desc,
                       lp_instance** out);
int lp_instance_destroy(lp_instance* inst);
/* Model descriptor the instance was created with. */
int lp_instance_model(lp_instance* inst, lp_model_desc* out);
/* Capture graphs for every (length, depth) of the grid — GraphGrid,
 * scheduler.hpp:21-32 — plus per-64-token chunk graphs (up to C_l = 512,
 * scheduler.hpp:46) for one-member standard launches. Each grid shape gets
 * variants chosen per batch at lp_submit (attention merge grid or not,
 * warp-MMA or tcgen05 attention); replays read every live size from device
 * metadata, so no variant depends on the histories. No-op when
 * use_graphs == 0. */
int lp_capture_graphs(lp_instance* inst, const int64_t* lengths, int32_t n_lengths,
                      const int32_t* depths, int32_t n_depths);

/* ---- the forward (replaces batch_service_time / packed_service_time) ----
 * members: `n` rows in plan order (sim.cpp:241-248); dummy pad rows implied
 * by shape->depth > n are never computed and never write KV.
 * token_ids: the packed new tokens of all members, sum(new_tokens) int32.
 * Asynchronous on the instance's stream. */
int lp_submit(lp_instance* inst, const lp_shape* shape, const lp_member* members, int32_t n,
              const int32_t* token_ids);
/* Block until the last submit finished; *service_ms = device time of the
 * forward (CUDA events on the instance stream). */
int lp_wait(lp_instance* inst, double* service_ms);
/* Ticketed form of lp_submit for pipelined / multi-instance drivers: the
 * forward is queued on the instance's stream and *ticket identifies it.
 * Metadata for up to 4 forwards can be staged ahead of the GPU; results (the
 * device time and the greedy first tokens, copied to pinned host memory at
 * the end of the forward) stay readable for the last 16 submits of the
 * instance — an older ticket is LP_ERR_STATE. lp_submit == lp_submit_async
 * with the ticket kept as "the last submit". */
int lp_submit_async(lp_instance* inst, const lp_shape* shape, const lp_member* members, int32_t n,
                    const int32_t* token_ids, int64_t* ticket);
/* *done = 1 once the forward and its first-token copy finished (cudaEventQuery;
 * never blocks). */
int lp_ticket_query(lp_instance* inst, int64_t ticket, int32_t* done);
/* Block until the ticket's forward finished; *service_ms = its device time. */
int lp_ticket_wait(lp_instance* inst, int64_t ticket, double* service_ms);
/* Greedy first tokens of the ticket's members (blocks until available). */
int lp_ticket_tokens(lp_instance* inst, int64_t ticket, int32_t* out, int32_t n);

/* Greedy first token (argmax of the last real token's logits) per member of
 * the last submit, in member order. */
int lp_read_next_tokens(lp_instance* inst, int32_t* out, int32_t n);
/* fp32 logits [n, vocab] of the last submit (debug/parity; large). */
int lp_read_logits(lp_instance* inst, float* out, size_t cap_floats);

/* Host->device bytes copied by the last lp_submit (token ids + metadata)
 * and device->host bytes of its result (the first tokens, copied at the end
 * of every forward). */
int lp_last_io(lp_instance* inst, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* Kernels the last lp_submit put on the GPU (graph kernel nodes or eager
 * launches): 1 + layers x (8 or 9) + 3. */
int lp_last_launches(lp_instance* inst, int32_t* kernels);
/* Device-side timing on the instance stream (CUDA events): record `slot`
 * (0..7); elapsed ms between two recorded slots (blocks on slot_b). */
int lp_timer_record(lp_instance* inst, int32_t slot);
int lp_timer_elapsed(lp_instance* inst, int32_t slot_a, int32_t slot_b, double* ms);

/* ---- paged KV cache ---- */
/* Page table of a session: up to `cap` page ids; *kv_len = resident tokens. */
int lp_session_pages(lp_instance* inst, int64_t session_id, int32_t* pages, int32_t cap,
                     int32_t* n_pages, int64_t* kv_len);
/* Free a finished session's pages. */
int lp_session_release(lp_instance* inst, int64_t session_id);
/* Copy K and V (bf16, [n, n_kv_heads, head_dim] each) of positions
 * [pos0, pos0+n) of one layer to host buffers. */
int lp_read_kv(lp_instance* inst, int64_t session_id, int32_t layer, int64_t pos0, int64_t n,
               uint16_t* k_out, uint16_t* v_out);
/* Move a session's KV to another instance (P2P over NVLink when the devices
 * differ). Asynchronous: the copy is ordered after the source's queued
 * forwards (event) and before the destination's next ones (its stream), and
 * the source's later work waits for the copy before reusing the pages. */
int lp_session_migrate(lp_instance* src, lp_instance* dst, int64_t session_id);
/* As lp_session_migrate, but the source keeps its copy (a session whose
 * long-prompt chunks are still running there while a later turn is served
 * elsewhere). */
int lp_session_copy(lp_instance* src, lp_instance* dst, int64_t session_id);

/* ---- deterministic synthetic inputs (shared with the CPU oracle) ---- */
/* token id of (seed, session, position): splitmix64 mix mod vocab. */
int32_t lp_synth_token(uint64_t seed, int64_t session_id, int64_t position, int32_t vocab);

const char* lp_last_error(void);
const char* lp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LAPS_PREFILL_H_ */
