// TEST INFRASTRUCTURE ONLY — the reference-oracle driver.
//
// Links the UNMODIFIED reference library compiled from
// /root/reference/proj/src/*.cpp (see oracle/Makefile) and exposes a tiny
// C ABI so tests and bench.py's reference arm can drive it through ctypes:
//
//   ref_simulate   — prefillsim `simulate` (tools/main.cpp:76-93): parse a
//                    config (config.cpp:116-145), apply `key=value` override
//                    lines (main.cpp:53-74), build_scenario + run_scenario
//                    (config.cpp:159, :374), write events.log / metrics.json
//                    (event_log.cpp:172, metrics.cpp:232).
//   ref_trace      — dump the synthetic request stream (build_workload,
//                    config.cpp:337) as text for the host-engine parity tests.
//   ref_service_ms — batch_service_time (cost_model.cpp:128-148).
//   ref_acceptance — run_acceptance (acceptance.cpp:899-928).
//
// Nothing in the product path loads this library.
#include <prefillsim/acceptance.hpp>
#include <prefillsim/config.hpp>
#include <prefillsim/cost_model.hpp>
#include <prefillsim/event_log.hpp>
#include <prefillsim/metrics.hpp>
#include <prefillsim/sim.hpp>

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>

using namespace prefillsim;

namespace {
std::string g_err;

ConfigMap make_map(const char* cfg_text, const char* overrides) {
  ConfigMap cfg = parse_config_text(cfg_text ? cfg_text : "");
  if (overrides && *overrides) {
    ConfigMap ov = parse_config_text(overrides);
    apply_overrides(cfg, ov);
  }
  return cfg;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Returns 0 on success. run_seconds gets the wall time of run_scenario
// (workload synthesis + engine run + metrics), n_dispatch the number of
// dispatch records.
int ref_simulate(const char* cfg_text, const char* overrides,
                 const char* out_dir, double* run_seconds,
                 int64_t* n_dispatch) {
  try {
    const ConfigMap cfg = make_map(cfg_text, overrides);
    const Scenario sc = build_scenario(cfg);
    const auto reqs = build_workload(sc);
    const auto t0 = std::chrono::steady_clock::now();
    RunResult rr = run(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid,
                       sc.ctrl);
    const auto t1 = std::chrono::steady_clock::now();
    if (run_seconds) *run_seconds = std::chrono::duration<double>(t1 - t0).count();
    if (n_dispatch) {
      int64_t n = 0;
      for (const auto& r : rr.log) n += r.kind == EventKind::kDispatch;
      *n_dispatch = n;
    }
    if (out_dir && *out_dir) {
      std::filesystem::create_directories(out_dir);
      write_event_log(std::string(out_dir) + "/events.log", rr.log);
      write_metrics(std::string(out_dir) + "/metrics.json", rr.report);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Writes "id session turn L H arrival(%.17g) deadline(%.17g|none)" lines.
int ref_trace(const char* cfg_text, const char* overrides, const char* path) {
  try {
    const ConfigMap cfg = make_map(cfg_text, overrides);
    const Scenario sc = build_scenario(cfg);
    const auto reqs = build_workload(sc);
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error("cannot write trace dump");
    for (const auto& r : reqs) {
      std::fprintf(f, "%" PRId64 " %" PRId64 " %d %" PRId64 " %" PRId64 " %.17g ",
                   r.id, r.session_id, r.turn, r.new_tokens, r.history_tokens,
                   r.arrival_ms);
      if (r.deadline_ms) std::fprintf(f, "%.17g\n", *r.deadline_ms);
      else std::fprintf(f, "none\n");
    }
    std::fclose(f);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double ref_service_ms(int64_t l_pad, int depth, int graph, const int64_t* L,
                      const int64_t* H, int n) {
  BatchShape s{l_pad, depth, graph ? ShapeKind::kGraph : ShapeKind::kStandard};
  std::vector<MemberShape> m;
  for (int i = 0; i < n; ++i) m.push_back({L[i], H[i]});
  try {
    return batch_service_time(s, m, CostParams{}, ExecOverheads{});
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

int ref_acceptance() {
  int bad = 0;
  for (const auto& r : run_acceptance()) {
    std::printf("c%d %s %s %s\n", r.id, r.name.c_str(), r.pass ? "PASS" : "FAIL",
                r.detail.c_str());
    bad += r.pass ? 0 : 1;
  }
  return bad;
}

}  // extern "C"

#ifdef REF_MAIN
// ref_sim <config-file|-> <out-dir> [key=value ...]
int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: ref_sim <config|-> <out-dir> [key=value...]\n");
    return 2;
  }
  std::string text;
  if (std::strcmp(argv[1], "-") != 0) {
    std::ifstream in(argv[1]);
    std::ostringstream ss;
    ss << in.rdbuf();
    text = ss.str();
  }
  std::string ov;
  for (int i = 3; i < argc; ++i) ov += std::string(argv[i]) + "\n";
  double secs = 0;
  int64_t nd = 0;
  if (ref_simulate(text.c_str(), ov.c_str(), argv[2], &secs, &nd) != 0) {
    std::fprintf(stderr, "error: %s\n", ref_last_error());
    return 1;
  }
  std::printf("dispatches %" PRId64 " run_s %.6f\n", nd, secs);
  return 0;
}
#endif
