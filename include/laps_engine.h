/*
 * laps_engine.h — C ABI of the host engine (dual queues, AWD batching,
 * length-bucket graph choice, temporal/spatial disaggregation, pool
 * controller). Replaces the reference's `prefillsim simulate`
 * (tools/main.cpp:76-93 -> config.cpp:159 build_scenario -> config.cpp:374
 * run_scenario -> sim.cpp:660 run) with one difference: every dispatch can
 * run its real forward on a B200 prefill instance (laps_prefill.h).
 *
 * Modes
 *   LP_SIM_COST_MODEL  service time = closed-form cost model; no GPU. The
 *                      events.log / metrics.json are byte-identical to the
 *                      reference's for the same config.
 *   LP_SIM_REPLAY      as above for the clock (so batch composition, queue
 *                      assignment, padding and chunking stay byte-identical),
 *                      and every dispatch ALSO executes on its GPU instance.
 *                      The engine does not wait for the GPU: forwards of
 *                      different instances run concurrently, measured times
 *                      are collected as they finish.
 *   LP_SIM_LIVE        virtual clock advanced by the measured GPU service time
 *                      of each forward (waits for every forward).
 *   LP_SIM_WALL        wall clock (steady_clock): arrivals are released in real
 *                      time, completions are the GPU's CUDA events, the
 *                      instances serve concurrently; TTFT includes engine,
 *                      H2D, launch and D2H time. With no instances the
 *                      forwards are emulated by sleeping for the cost-model
 *                      service time (host-side tests of the wall clock).
 */
#ifndef LAPS_ENGINE_H_
#define LAPS_ENGINE_H_

#include <stdint.h>

#include "laps_prefill.h"

#ifdef __cplusplus
extern "C" {
#endif

#define LP_SIM_COST_MODEL 0
#define LP_SIM_REPLAY 1
#define LP_SIM_LIVE 2
#define LP_SIM_WALL 3

typedef struct lp_sim_stats {
  int64_t arrivals;
  int64_t completed;
  int64_t dispatches;
  int64_t gpu_forwards;      /* forwards executed on GPU (excl. history fills) */
  int64_t fill_forwards;     /* history fills for non-resident KV */
  int64_t kv_migrations;     /* sessions moved between instances */
  int64_t real_tokens;       /* new tokens computed by dispatched forwards */
  double active_ms;          /* metrics.json active_ms (engine clock) */
  double ttft_mean_ms, ttft_p50_ms, ttft_p90_ms, ttft_p99_ms;
  double rps;                /* completions per second of active interval */
  double slo_violation;
  double gpu_ms_total;       /* sum of measured forward times */
  double engine_wall_s;      /* host wall time of the whole run */
  /* Timed window (lp_sim_opts); zero when no window was requested. */
  int64_t window_dispatches;  /* engine dispatches executed inside the window */
  int64_t window_requests;    /* requests whose final forward is in the window */
  int64_t window_fills;       /* history-fill forwards inside the window */
  int64_t window_kernels;     /* kernels the window's forwards launched */
  int64_t window_h2d_bytes;   /* token ids + metadata copied host->device */
  int64_t window_d2h_bytes;   /* first tokens copied device->host */
  double window_device_ms;    /* max over instances: CUDA-event time from
                                 before the window's first forward to after
                                 its last one, on each instance's stream */
  double window_wall_ms;      /* host steady_clock from the first window
                                 submit until every window forward finished
                                 and its first tokens were read on the host */
} lp_sim_stats;

/* Run options (all zero = lp_sim_run). */
typedef struct lp_sim_opts {
  int64_t window_first;  /* GPU dispatches [first, first + count) form the  */
  int64_t window_count;  /* timed window (REPLAY mode); 0 = no window      */
  int32_t stop_after_window;  /* 1: later dispatches run on the clock only  */
  int32_t reserved;
} lp_sim_opts;

/* Run a scenario. cfg_text / overrides: `key = value` lines (reference key
 * names). out_dir: if non-empty, events.log + metrics.json (+ forwards.csv
 * when a GPU ran) are written there. insts: n_insts GPU instances (sim
 * instance i runs on insts[i % n_insts]); may be NULL for the cost model.
 * token_seed: seed of the synthetic token ids (lp_synth_token). */
int lp_sim_run(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
               lp_instance** insts, int32_t n_insts, uint64_t token_seed, lp_sim_stats* stats);

/* lp_sim_run with options (a timed window of dispatches for benchmarks). */
int lp_sim_run_ex(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
                  lp_instance** insts, int32_t n_insts, uint64_t token_seed, const lp_sim_opts* opts,
                  lp_sim_stats* stats);

/* The reference CLI's `prefillsim sweep --param P --values v1,v2,...`
 * (tools/main.cpp:114-168): for each value (sorted ascending) apply
 * apply_sweep_param (config.cpp:353-372) to a fresh copy of the config, run the
 * engine in `mode` (cost model, or on the GPU instances), and write
 * out_dir/sweep.csv with the reference's columns and number formats. */
int lp_sim_sweep(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
                 lp_instance** insts, int32_t n_insts, uint64_t token_seed, const char* param,
                 const char* values_csv);

/* Dump the scenario's request stream as text lines
 * "id session turn L H arrival(%.17g) deadline(%.17g|none)". */
int lp_sim_trace(const char* cfg_text, const char* overrides, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* LAPS_ENGINE_H_ */
