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
//   ref_sweep      — the CLI's `sweep` (tools/main.cpp:114-168) restated on
//                    the library's apply_sweep_param / run_scenario.
//
// Nothing in the product path loads this library.
#include <prefillsim/acceptance.hpp>
#include <prefillsim/config.hpp>
#include <prefillsim/cost_model.hpp>
#include <prefillsim/event_log.hpp>
#include <prefillsim/metrics.hpp>
#include <prefillsim/sim.hpp>

#include <algorithm>
#include <chrono>
#include <vector>
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

// ref_sweep — restates the reference CLI's `sweep` subcommand
// (tools/main.cpp:114-168; the CLI itself needs CLI11, absent here) on top of
// the reference library's apply_sweep_param / build_scenario / run_scenario
// (config.cpp:353-378): same value order, columns and printf formats.
int ref_sweep(const char* cfg_text, const char* overrides, const char* out_dir, const char* param,
              const char* values_csv) {
  try {
    const ConfigMap base = make_map(cfg_text, overrides);
    std::vector<double> values;
    std::stringstream ss(values_csv ? values_csv : "");
    std::string item;
    while (std::getline(ss, item, ',')) {
      if (item.empty()) continue;
      values.push_back(std::stod(item));
    }
    if (values.empty()) throw std::runtime_error("empty values");
    std::sort(values.begin(), values.end());
    auto cls = [](std::string& row, const ClassMetrics& c) {
      char buf[256];
      std::snprintf(buf, sizeof buf, ",%lld,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%lld,%.6f,%.6f,%.6f",
                    static_cast<long long>(c.completed), c.ttft_mean_ms, c.ttft_p50_ms, c.ttft_p90_ms,
                    c.ttft_p99_ms, c.rps, c.slo_violation, c.mean_wait_ms, static_cast<long long>(c.batches),
                    c.mean_depth, c.graph_hit_rate, c.padding_overhead);
      row += buf;
    };
    const char* cols_all =
        "completed,ttft_mean_ms,ttft_p50_ms,ttft_p90_ms,ttft_p99_ms,rps,slo_violation,mean_wait_ms,batches,"
        "mean_depth,graph_hit_rate,padding_overhead";
    std::string csv = "param,value,arrivals,active_ms,migrations";
    for (const char* scope : {"overall_", "short_", "long_"}) {
      std::stringstream cols(cols_all);
      std::string col;
      while (std::getline(cols, col, ',')) csv += std::string(",") + scope + col;
    }
    csv += '\n';
    for (double v : values) {
      ConfigMap cfg = base;
      apply_sweep_param(cfg, param, v);
      const RunResult rr = run_scenario(build_scenario(cfg));
      char head[160];
      std::snprintf(head, sizeof head, "%s,%.6f,%lld,%.6f,%lld", param, v,
                    static_cast<long long>(rr.report.arrivals), rr.report.active_ms,
                    static_cast<long long>(rr.report.migrations));
      std::string row = head;
      cls(row, rr.report.overall);
      cls(row, rr.report.short_cls);
      cls(row, rr.report.long_cls);
      csv += row + '\n';
    }
    std::filesystem::create_directories(out_dir);
    std::ofstream os(std::string(out_dir) + "/sweep.csv", std::ios::binary);
    os << csv;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
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
