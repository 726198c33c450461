// ForwardBackend that runs every dispatched batch on a B200 prefill instance
// through the public C ABI (laps_prefill.h), plus the engine's own C ABI
// (laps_engine.h).
//
// Session KV residency: a member (session, L, H) needs positions [0, H) on
// the instance that runs it. If another instance holds them, the pages move
// over NVLink (lp_session_migrate); positions nobody computed (trace
// gen_tokens, a later turn dispatched before its predecessor) are produced by
// a deterministic history fill forward over the synthetic token ids. A
// session's pages are released after its last turn's final forward.
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <filesystem>
#include <memory>
#include <fstream>
#include <sstream>
#include <unordered_map>

#include "../../../include/laps_engine.h"
#include "laps_host.hpp"

namespace laps {

namespace {

void check(int rc, const char* what) {
  if (rc != LP_OK) throw std::runtime_error(std::string(what) + ": " + lp_last_error());
}

class GpuBackend final : public ForwardBackend {
 public:
  GpuBackend(lp_instance** insts, int n, bool live, uint64_t token_seed, int32_t vocab,
             const std::vector<Request>& reqs)
      : insts_(insts, insts + n), live_(live), seed_(token_seed), vocab_(vocab) {
    for (const auto& r : reqs) {
      auto& last = last_turn_[r.session_id];
      last = std::max(last, r.turn);
      turn_of_[r.id] = r.turn;
    }
  }

  double forward(const ForwardCall& call) override {
    const int gi = call.inst % static_cast<int>(insts_.size());
    lp_instance* inst = insts_[static_cast<size_t>(gi)];
    for (const auto& row : call.rows) make_resident(gi, row.session_id, row.history);

    std::vector<lp_member> mem;
    std::vector<int32_t> toks;
    for (const auto& row : call.rows) {
      mem.push_back(lp_member{row.req_id, row.session_id, row.new_tokens, row.history, 1, 0});
      for (Tokens p = row.history; p < row.history + row.new_tokens; ++p)
        toks.push_back(lp_synth_token(seed_, row.session_id, p, vocab_));
    }
    lp_shape shape{call.shape.l_pad, call.shape.depth,
                   call.kind == ForwardKind::kPacked       ? LP_KIND_PACKED
                   : call.shape.kind == ShapeKind::kGraph ? LP_KIND_GRAPH
                                                          : LP_KIND_STANDARD};
    check(lp_submit(inst, &shape, mem.data(), static_cast<int32_t>(mem.size()), toks.data()), "lp_submit");
    double ms = 0;
    check(lp_wait(inst, &ms), "lp_wait");
    first_tok_.resize(mem.size());
    check(lp_read_next_tokens(inst, first_tok_.data(), static_cast<int32_t>(mem.size())), "next tokens");

    for (const auto& row : call.rows) {
      owner_[row.session_id] = gi;
      if (row.finishes_request) {
        first_token_[row.req_id] = first_tok_[&row - call.rows.data()];
        if (turn_of_[row.req_id] >= last_turn_[row.session_id]) {
          check(lp_session_release(inst, row.session_id), "release");
          owner_.erase(row.session_id);
        }
      }
    }
    stats_.gpu_forwards += 1;
    stats_.gpu_ms_total += ms;
    Tokens t = 0, hist = 0;
    double pairs = 0;  // attention (query, key) pairs: sum L (H + (L + 1) / 2)
    for (const auto& row : call.rows) {
      t += row.new_tokens;
      hist += row.history;
      pairs += static_cast<double>(row.new_tokens) * (static_cast<double>(row.history) + (row.new_tokens + 1) / 2.0);
    }
    stats_.real_tokens += t;
    log_ << call.inst << ',' << static_cast<int>(call.kind) << ',' << call.shape.l_pad << ','
         << call.shape.depth << ',' << (call.shape.kind == ShapeKind::kGraph ? 1 : 0) << ',' << call.rows.size()
         << ',' << t << ',' << hist << ',' << pairs << ',' << call.model_service_ms << ',' << ms << '\n';
    return live_ ? ms : call.model_service_ms;
  }

  void write(const std::string& dir) const {
    std::ofstream f(dir + "/forwards.csv");
    f << "inst,kind,l_pad,depth,graph,members,tokens,hist_tokens,attn_pairs,model_ms,gpu_ms\n" << log_.str();
    std::ofstream g(dir + "/first_tokens.csv");
    g << "req,token\n";
    std::vector<std::pair<RequestId, int32_t>> v(first_token_.begin(), first_token_.end());
    std::sort(v.begin(), v.end());
    for (auto& [r, t] : v) g << r << ',' << t << '\n';
  }

  // Sessions still resident when the run ends (their last turn did not
  // finish inside the simulated window) are released, so an instance reused
  // for the next run (sweeps, repeated benchmarks) starts from an empty pool:
  // session ids restart at 0 in every workload.
  ~GpuBackend() override {
    for (const auto& [sid, gi] : owner_) lp_session_release(insts_[static_cast<size_t>(gi)], sid);
  }

  lp_sim_stats stats_{};

 private:
  int64_t resident(int gi, std::int64_t sid) {
    int32_t np = 0;
    int64_t kv = 0;
    check(lp_session_pages(insts_[static_cast<size_t>(gi)], sid, nullptr, 0, &np, &kv), "pages");
    return kv;
  }

  void make_resident(int gi, std::int64_t sid, Tokens H) {
    if (H == 0) return;
    int64_t have = resident(gi, sid);
    if (have >= H) return;
    auto it = owner_.find(sid);
    if (it != owner_.end() && it->second != gi && resident(it->second, sid) > have) {
      check(lp_session_migrate(insts_[static_cast<size_t>(it->second)], insts_[static_cast<size_t>(gi)], sid),
            "migrate");
      stats_.kv_migrations += 1;
      owner_[sid] = gi;
      have = resident(gi, sid);
      if (have >= H) return;
    }
    // Deterministic fill of the missing positions [have, H).
    lp_instance* inst = insts_[static_cast<size_t>(gi)];
    constexpr Tokens kFill = 2048;
    for (Tokens p = have; p < H; p += kFill) {
      const Tokens n = std::min(kFill, H - p);
      lp_member m{-1, sid, n, p, 0, 0};
      std::vector<int32_t> toks;
      for (Tokens q = p; q < p + n; ++q) toks.push_back(lp_synth_token(seed_, sid, q, vocab_));
      lp_shape shape{n, 1, LP_KIND_STANDARD};
      check(lp_submit(inst, &shape, &m, 1, toks.data()), "fill submit");
      double ms = 0;
      check(lp_wait(inst, &ms), "fill wait");
      stats_.fill_forwards += 1;
    }
    owner_[sid] = gi;
  }

  std::vector<lp_instance*> insts_;
  bool live_;
  uint64_t seed_;
  int32_t vocab_;
  std::unordered_map<std::int64_t, int> last_turn_;
  std::unordered_map<RequestId, int> turn_of_;
  std::unordered_map<std::int64_t, int> owner_;
  std::unordered_map<RequestId, int32_t> first_token_;
  std::vector<int32_t> first_tok_;
  std::ostringstream log_;
};

ConfigMap config_from(const char* cfg_text, const char* overrides) {
  ConfigMap cfg = parse_config_text(cfg_text ? cfg_text : "");
  if (overrides && *overrides) apply_overrides(cfg, parse_config_text(overrides));
  return cfg;
}

Scenario scenario_from(const char* cfg_text, const char* overrides) {
  return build_scenario(config_from(cfg_text, overrides));
}

// One engine run: closed-form service times, or every dispatch on the GPU
// instances (replay: cost-model clock; live: measured clock).
RunResult run_mode(const Scenario& sc, int32_t mode, lp_instance** insts, int32_t n_insts, uint64_t token_seed,
                   std::unique_ptr<GpuBackend>* keep) {
  const std::vector<Request> reqs = build_workload(sc);
  if (mode == LP_SIM_COST_MODEL) return run(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl);
  if (!insts || n_insts < 1) throw ConfigError("GPU modes need at least one instance");
  lp_model_desc md{};
  check(lp_instance_model(insts[0], &md), "lp_instance_model");
  auto gpu = std::make_unique<GpuBackend>(insts, n_insts, mode == LP_SIM_LIVE, token_seed, md.vocab, reqs);
  RunResult rr = run_with_backend(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl, *gpu);
  if (keep) *keep = std::move(gpu);
  return rr;
}

// sweep.csv row columns of the reference CLI (tools/main.cpp:97-113).
void csv_class(std::string& row, const ClassMetrics& c) {
  char buf[256];
  std::snprintf(buf, sizeof buf, ",%lld,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%lld,%.6f,%.6f,%.6f",
                static_cast<long long>(c.completed), c.ttft_mean_ms, c.ttft_p50_ms, c.ttft_p90_ms, c.ttft_p99_ms,
                c.rps, c.slo_violation, c.mean_wait_ms, static_cast<long long>(c.batches), c.mean_depth,
                c.graph_hit_rate, c.padding_overhead);
  row += buf;
}

}  // namespace
}  // namespace laps

namespace lp {
void set_last_error(const std::string& msg);  // shared with laps_prefill.h's lp_last_error()
}

extern "C" {

int lp_sim_run(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
               lp_instance** insts, int32_t n_insts, uint64_t token_seed, lp_sim_stats* stats) {
  using namespace laps;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const Scenario sc = scenario_from(cfg_text, overrides);
    lp_sim_stats st{};
    std::unique_ptr<GpuBackend> gpu;
    RunResult rr = run_mode(sc, mode, insts, n_insts, token_seed, &gpu);
    if (gpu) st = gpu->stats_;
    if (out_dir && *out_dir) {
      std::filesystem::create_directories(out_dir);
      write_event_log(std::string(out_dir) + "/events.log", rr.log);
      write_metrics(std::string(out_dir) + "/metrics.json", rr.report);
      if (gpu) gpu->write(out_dir);
    }
    if (stats) {
      st.arrivals = rr.report.arrivals;
      st.completed = rr.report.overall.completed;
      st.dispatches = std::count_if(rr.log.begin(), rr.log.end(),
                                    [](const LogRecord& r) { return r.kind == EventKind::kDispatch; });
      st.active_ms = rr.report.active_ms;
      st.ttft_mean_ms = rr.report.overall.ttft_mean_ms;
      st.ttft_p50_ms = rr.report.overall.ttft_p50_ms;
      st.ttft_p90_ms = rr.report.overall.ttft_p90_ms;
      st.ttft_p99_ms = rr.report.overall.ttft_p99_ms;
      st.rps = rr.report.overall.rps;
      st.slo_violation = rr.report.overall.slo_violation;
      st.engine_wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      *stats = st;
    }
    return LP_OK;
  } catch (const laps::ShapeMismatch& e) {
    lp::set_last_error(e.what());
    return LP_ERR_SHAPE;
  } catch (const laps::ConfigError& e) {
    lp::set_last_error(e.what());
    return LP_ERR_CONFIG;
  } catch (const std::exception& e) {
    lp::set_last_error(e.what());
    return LP_ERR_INTERNAL;
  }
}

int lp_sim_sweep(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
                 lp_instance** insts, int32_t n_insts, uint64_t token_seed, const char* param,
                 const char* values_csv) {
  using namespace laps;
  try {
    if (!param || !*param) throw ConfigError("sweep: empty parameter name");
    const ConfigMap base = config_from(cfg_text, overrides);
    std::vector<double> values;
    std::stringstream ss(values_csv ? values_csv : "");
    std::string item;
    while (std::getline(ss, item, ',')) {
      if (item.empty()) continue;
      values.push_back(std::stod(item));
    }
    if (values.empty()) throw ConfigError("sweep: --values parsed to an empty list");
    std::sort(values.begin(), values.end());
    static const char* kClassCols =
        "completed,ttft_mean_ms,ttft_p50_ms,ttft_p90_ms,ttft_p99_ms,rps,slo_violation,mean_wait_ms,batches,"
        "mean_depth,graph_hit_rate,padding_overhead";
    std::string csv = "param,value,arrivals,active_ms,migrations";
    for (const char* scope : {"overall_", "short_", "long_"}) {
      std::stringstream cols(kClassCols);
      std::string col;
      while (std::getline(cols, col, ',')) csv += std::string(",") + scope + col;
    }
    csv += '\n';
    for (double v : values) {
      ConfigMap cfg = base;  // fresh copy: scaling params read base values
      apply_sweep_param(cfg, param, v);
      const RunResult rr = run_mode(build_scenario(cfg), mode, insts, n_insts, token_seed, nullptr);
      char head[160];
      std::snprintf(head, sizeof head, "%s,%.6f,%lld,%.6f,%lld", param, v,
                    static_cast<long long>(rr.report.arrivals), rr.report.active_ms,
                    static_cast<long long>(rr.report.migrations));
      std::string row = head;
      csv_class(row, rr.report.overall);
      csv_class(row, rr.report.short_cls);
      csv_class(row, rr.report.long_cls);
      csv += row + '\n';
    }
    std::filesystem::create_directories(out_dir);
    std::ofstream os(std::string(out_dir) + "/sweep.csv", std::ios::binary);
    if (!os) throw std::runtime_error("sweep: cannot write sweep.csv");
    os << csv;
    return LP_OK;
  } catch (const laps::ConfigError& e) {
    lp::set_last_error(e.what());
    return LP_ERR_CONFIG;
  } catch (const std::exception& e) {
    lp::set_last_error(e.what());
    return LP_ERR_INTERNAL;
  }
}

int lp_sim_trace(const char* cfg_text, const char* overrides, const char* path) {
  using namespace laps;
  try {
    const auto reqs = build_workload(scenario_from(cfg_text, overrides));
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::runtime_error("cannot write trace dump");
    for (const auto& r : reqs) {
      std::fprintf(f, "%" PRId64 " %" PRId64 " %d %" PRId64 " %" PRId64 " %.17g ", r.id, r.session_id, r.turn,
                   r.new_tokens, r.history_tokens, r.arrival_ms);
      if (r.deadline_ms) std::fprintf(f, "%.17g\n", *r.deadline_ms);
      else std::fprintf(f, "none\n");
    }
    std::fclose(f);
    return LP_OK;
  } catch (const std::exception& e) {
    lp::set_last_error(e.what());
    return LP_ERR_CONFIG;
  }
}

}  // extern "C"
