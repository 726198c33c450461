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
 *                      and every dispatch ALSO executes on its GPU instance;
 *                      measured forward times are reported alongside.
 *   LP_SIM_LIVE        the clock advances by the measured GPU service time:
 *                      real TTFT / req/s of the B200 path under the policy.
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
} lp_sim_stats;

/* Run a scenario. cfg_text / overrides: `key = value` lines (reference key
 * names). out_dir: if non-empty, events.log + metrics.json (+ forwards.csv
 * when a GPU ran) are written there. insts: n_insts GPU instances (sim
 * instance i runs on insts[i % n_insts]); may be NULL for the cost model.
 * token_seed: seed of the synthetic token ids (lp_synth_token). */
int lp_sim_run(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
               lp_instance** insts, int32_t n_insts, uint64_t token_seed, lp_sim_stats* stats);

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
