/*
 * laps_simulate.c — the reference's `prefillsim simulate --config <cfg> --out <dir>`
 * (tools/main.cpp:76-93) driven through this repo's two C ABIs from plain C,
 * the way a C / C++ / Go (cgo) / Java (JNI) host binds liblaps_prefill.so:
 *
 *   laps_simulate <config file> <out dir> [cost|replay|live] [tiny|7b|32b]
 *
 *   cost    closed-form service times (reference semantics, no GPU);
 *   replay  cost-model clock, every dispatch also runs on the B200 instance
 *           (events.log byte-identical to `cost`);
 *   live    the clock advances by the measured GPU forward times.
 *
 * Prints the run statistics (lp_sim_stats) as one JSON line.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "laps_engine.h"
#include "laps_prefill.h"

static char* slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc((size_t)n + 1);
  if (buf && fread(buf, 1, (size_t)n, f) != (size_t)n) {
    free(buf);
    buf = NULL;
  }
  if (buf) buf[n] = 0;
  fclose(f);
  return buf;
}

static lp_model_desc model_of(const char* name) {
  /* Qwen2.5 shapes (random-init weights, seed 1234) and the tiny test decoder. */
  lp_model_desc m = {256, 704, 2, 4, 2, 64, 1024, 1e6f, 1e-6f, 0.02f, 1234};
  if (strcmp(name, "7b") == 0) {
    lp_model_desc q = {3584, 18944, 28, 28, 4, 128, 152064, 1e6f, 1e-6f, 0.02f, 1234};
    m = q;
  } else if (strcmp(name, "32b") == 0) {
    lp_model_desc q = {5120, 27648, 64, 40, 8, 128, 152064, 1e6f, 1e-6f, 0.02f, 1234};
    m = q;
  }
  return m;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: %s <config> <out dir> [cost|replay|live] [tiny|7b|32b]\n", argv[0]);
    return 2;
  }
  const char* mode_s = argc > 3 ? argv[3] : "cost";
  const char* model_s = argc > 4 ? argv[4] : "tiny";
  const int mode = strcmp(mode_s, "live") == 0 ? LP_SIM_LIVE : strcmp(mode_s, "replay") == 0 ? LP_SIM_REPLAY
                                                                                            : LP_SIM_COST_MODEL;
  char* cfg = slurp(argv[1]);
  if (!cfg) {
    fprintf(stderr, "cannot read %s\n", argv[1]);
    return 2;
  }
  lp_instance* inst = NULL;
  if (mode != LP_SIM_COST_MODEL) {
    const lp_model_desc md = model_of(model_s);
    const lp_instance_desc d = {/*device*/ 0, /*page_size*/ 64, /*kv_pages*/ 0, /*max_tokens*/ 16384,
                                /*max_members*/ 64, /*use_graphs*/ 1};
    if (lp_instance_create(&md, &d, &inst) != LP_OK) {
      fprintf(stderr, "lp_instance_create: %s\n", lp_last_error());
      return 1;
    }
    /* GraphGrid defaults (scheduler.hpp:21-32): 6 lengths x 7 depths. */
    const int64_t lens[] = {8, 16, 32, 64, 128, 256};
    const int32_t deps[] = {1, 2, 4, 8, 16, 32, 64};
    if (lp_capture_graphs(inst, lens, 6, deps, 7) != LP_OK) {
      fprintf(stderr, "lp_capture_graphs: %s\n", lp_last_error());
      return 1;
    }
  }
  lp_sim_stats st;
  memset(&st, 0, sizeof st);
  const int rc = lp_sim_run(cfg, "", argv[2], mode, inst ? &inst : NULL, inst ? 1 : 0, 7, &st);
  if (rc != LP_OK) {
    fprintf(stderr, "lp_sim_run: %s\n", lp_last_error());
    return 1; /* the reference CLI maps ConfigError / ShapeMismatch to exit code 1 (main.cpp:273-276) */
  }
  printf("{\"mode\": \"%s\", \"arrivals\": %lld, \"completed\": %lld, \"dispatches\": %lld, \"gpu_forwards\": %lld, "
         "\"ttft_p50_ms\": %.6f, \"ttft_p90_ms\": %.6f, \"rps\": %.6f, \"slo_violation\": %.6f, "
         "\"gpu_ms_total\": %.6f}\n",
         mode_s, (long long)st.arrivals, (long long)st.completed, (long long)st.dispatches,
         (long long)st.gpu_forwards, st.ttft_p50_ms, st.ttft_p90_ms, st.rps, st.slo_violation, st.gpu_ms_total);
  if (inst) lp_instance_destroy(inst);
  free(cfg);
  return 0;
}
