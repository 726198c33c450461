// The tier on B200 instances: a ForwardBackend that queues every dispatched
// forward on its lane's GPU through the public C ABI (laps_prefill.h) without
// waiting for it, plus the engine's own C ABI (laps_engine.h).
//
//   Sessions   a member (session, L, H) needs positions [0, H) on the GPU
//              that runs it. The session book knows which instances hold a
//              session; KV moves over NVLink (lp_session_migrate, or
//              lp_session_copy while a long prompt is still chunking on the
//              source), positions nobody computed yet (trace gen_tokens, a
//              later turn served before its predecessor) are produced by a
//              deterministic fill forward. Every copy is released once all of
//              the session's turns in the stream have finished.
//   Tickets    each forward returns a ticket; results (device ms, greedy
//              first tokens) are collected when the engine's clock needs them
//              (LIVE), when they finish (WALL), or lazily before the
//              instance's ticket ring wraps (REPLAY), so up to ~12 forwards
//              per GPU are queued ahead and N GPUs run concurrently.
//   Window     benchmarks time a contiguous range of dispatches with CUDA
//              events on every instance (device time) and steady_clock
//              (end to end, H2D + forwards + first-token reads).
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <memory>
#include <set>
#include <sstream>
#include <unordered_map>

#include <nvtx3/nvToolsExt.h>

#include "../../../include/laps_engine.h"
#include "laps_host.hpp"

namespace lp {
void set_last_error(const std::string& msg);  // shared with laps_prefill.h's lp_last_error()
}

namespace laps {

namespace {

void ok(int rc, const char* what) {
  if (rc != LP_OK) throw std::runtime_error(std::string(what) + ": " + lp_last_error());
}

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); }

// One executed forward (engine dispatch or history fill).
struct Forward {
  int gpu = 0;
  std::int64_t ticket = -1;
  bool fill = false;
  bool harvested = false;
  bool in_window = false;
  ForwardCall call;       // engine dispatches only
  double gpu_ms = 0;
  Tokens tokens = 0, hist = 0;
  double pairs = 0;       // attention (query, key) pairs: sum L (H + (L + 1) / 2)
  std::vector<int32_t> first;  // greedy first token per member
};

class GpuTier final : public ForwardBackend {
 public:
  GpuTier(lp_instance** insts, int n, int32_t mode, uint64_t token_seed, int32_t vocab,
          const std::vector<Request>& reqs, const lp_sim_opts& opts)
      : gpus_(insts, insts + n), mode_(mode), seed_(token_seed), vocab_(vocab), opts_(opts), pending_(gpus_.size()),
        next_ticket_(gpus_.size(), 0) {
    for (const Request& r : reqs) turns_[r.session_id] += 1;
  }

  ~GpuTier() override {
    // Sessions whose last turn fell outside the run: free every copy, so an
    // instance reused for the next run starts from an empty pool.
    for (auto& [sid, where] : holders_)
      for (int g : where) lp_session_release(gpus_[static_cast<size_t>(g)], sid);
  }

  // ---- ForwardBackend
  std::uint64_t launch(const ForwardCall& call) override {
    const std::int64_t k = dispatches_++;
    const bool before = opts_.window_count > 0 && k < opts_.window_first;
    const bool inside = opts_.window_count > 0 && k >= opts_.window_first &&
                        k < opts_.window_first + opts_.window_count;
    if (opts_.window_count > 0 && !before && !inside && opts_.stop_after_window) return 0;  // clock only
    if (inside && k == opts_.window_first) open_window();
    char tag[96];  // NVTX: one range per engine dispatch (profilers: --nvtx-include "dispatch*")
    std::snprintf(tag, sizeof tag, "dispatch %lld lane %d %s %lldx%d", static_cast<long long>(k), call.inst,
                  call.kind == ForwardKind::kLongChunk ? "chunk" : call.kind == ForwardKind::kPacked ? "packed" : "batch",
                  static_cast<long long>(call.shape.l_pad), call.shape.depth);
    nvtxRangePushA(tag);
    struct Pop {
      ~Pop() { nvtxRangePop(); }
    } pop;
    const int g = call.inst % static_cast<int>(gpus_.size());
    for (const ForwardRow& row : call.rows) make_resident(g, row.session_id, row.history, inside);

    std::vector<lp_member> members;
    std::vector<int32_t> toks;
    Forward f;
    f.gpu = g;
    f.in_window = inside;
    for (const ForwardRow& row : call.rows) {
      // Only a request's final forward needs the LM head (its first token).
      members.push_back(lp_member{row.req_id, row.session_id, row.new_tokens, row.history,
                                  row.finishes_request ? 1 : 0, 0});
      for (Tokens p = row.history; p < row.history + row.new_tokens; ++p)
        toks.push_back(lp_synth_token(seed_, row.session_id, p, vocab_));
      f.tokens += row.new_tokens;
      f.hist += row.history;
      f.pairs += static_cast<double>(row.new_tokens) *
                 (static_cast<double>(row.history) + static_cast<double>(row.new_tokens + 1) / 2.0);
    }
    const lp_shape shape{call.shape.l_pad, call.shape.depth,
                         call.kind == ForwardKind::kPacked       ? LP_KIND_PACKED
                         : call.shape.kind == ShapeKind::kGraph ? LP_KIND_GRAPH
                                                                : LP_KIND_STANDARD};
    f.call = call;
    const size_t idx = submit(f, shape, members.data(), static_cast<int32_t>(members.size()), toks.data());
    after_forward(g, call);
    stats_.gpu_forwards += 1;
    stats_.real_tokens += f.tokens;
    if (inside) {
      win_.dispatches += 1;
      for (const ForwardRow& row : call.rows) win_.requests += row.finishes_request ? 1 : 0;
      if (k == opts_.window_first + opts_.window_count - 1) close_window();
    }
    return idx + 1;
  }

  double clock_ms(std::uint64_t handle, const ForwardCall& call) override {
    if (mode_ != LP_SIM_LIVE || handle == 0) return call.model_service_ms;
    Forward& f = log_[handle - 1];
    harvest(f);
    return f.gpu_ms;
  }

  bool poll(std::uint64_t handle, double* service_ms) override {
    Forward& f = log_[handle - 1];
    if (!f.harvested) {
      int32_t done = 0;
      ok(lp_ticket_query(gpus_[static_cast<size_t>(f.gpu)], f.ticket, &done), "lp_ticket_query");
      if (!done) return false;
      harvest(f);
    }
    *service_ms = f.gpu_ms;
    return true;
  }

  void finish_run() override {
    for (Forward& f : log_) harvest(f);
  }

  void write(const std::string& dir) const {
    std::ofstream out(dir + "/forwards.csv");
    out << "inst,kind,l_pad,depth,graph,members,tokens,hist_tokens,attn_pairs,model_ms,gpu_ms,window,finished\n";
    std::ofstream first(dir + "/first_tokens.csv");
    first << "req,token\n";
    std::vector<std::pair<RequestId, int32_t>> firsts;
    for (const Forward& f : log_) {
      if (f.fill) continue;
      const ForwardCall& c = f.call;
      out << c.inst << ',' << static_cast<int>(c.kind) << ',' << c.shape.l_pad << ',' << c.shape.depth << ','
          << (c.shape.kind == ShapeKind::kGraph ? 1 : 0) << ',' << c.rows.size() << ',' << f.tokens << ','
          << f.hist << ',' << f.pairs << ',' << c.model_service_ms << ',' << f.gpu_ms << ',' << (f.in_window ? 1 : 0)
          << ',' << std::count_if(c.rows.begin(), c.rows.end(), [](const ForwardRow& r) { return r.finishes_request; })
          << '\n';
      for (size_t i = 0; i < c.rows.size() && i < f.first.size(); ++i)
        if (c.rows[i].finishes_request) firsts.emplace_back(c.rows[i].req_id, f.first[i]);
    }
    std::sort(firsts.begin(), firsts.end());
    for (auto& [r, t] : firsts) first << r << ',' << t << '\n';
  }

  void fill_stats(lp_sim_stats& st) const {
    st.gpu_forwards = stats_.gpu_forwards;
    st.fill_forwards = stats_.fill_forwards;
    st.kv_migrations = stats_.kv_migrations;
    st.real_tokens = stats_.real_tokens;
    double total = 0;
    for (const Forward& f : log_)
      if (!f.fill) total += f.gpu_ms;
    st.gpu_ms_total = total;
    st.window_dispatches = win_.dispatches;
    st.window_requests = win_.requests;
    st.window_fills = win_.fills;
    st.window_kernels = win_.kernels;
    st.window_h2d_bytes = win_.h2d;
    st.window_d2h_bytes = win_.d2h;
    st.window_device_ms = win_.device_ms;
    st.window_wall_ms = win_.wall_ms;
  }

 private:
  // Queue one forward; collects old results first so the instance's ticket
  // ring (16 results) never drops one we still need.
  size_t submit(Forward f, const lp_shape& shape, const lp_member* m, int32_t n, const int32_t* toks) {
    lp_instance* inst = gpus_[static_cast<size_t>(f.gpu)];
    auto& queue = pending_[static_cast<size_t>(f.gpu)];
    // Collect by AGE, not by count: forwards the engine polls are harvested
    // out of order, so a fill could otherwise outlive the instance's ticket
    // ring. Tickets are issued in order per instance, so the queue (submit
    // order) has its oldest entry in front.
    const std::int64_t next = next_ticket_[static_cast<size_t>(f.gpu)];
    while (!queue.empty() && log_[queue.front()].ticket + static_cast<std::int64_t>(kAhead) <= next)
      harvest(log_[queue.front()]);
    ok(lp_submit_async(inst, &shape, m, n, toks, &f.ticket), "lp_submit_async");
    next_ticket_[static_cast<size_t>(f.gpu)] = f.ticket + 1;
    if (f.in_window) {
      int32_t kernels = 0;
      int64_t h2d = 0, d2h = 0;
      ok(lp_last_launches(inst, &kernels), "lp_last_launches");
      ok(lp_last_io(inst, &h2d, &d2h), "lp_last_io");
      win_.kernels += kernels;
      win_.h2d += h2d;
      win_.d2h += d2h;
    }
    log_.push_back(std::move(f));
    queue.push_back(log_.size() - 1);
    return log_.size() - 1;
  }

  void harvest(Forward& f) {
    if (f.harvested) return;
    lp_instance* inst = gpus_[static_cast<size_t>(f.gpu)];
    ok(lp_ticket_wait(inst, f.ticket, &f.gpu_ms), "lp_ticket_wait");
    if (!f.fill) {
      f.first.resize(f.call.rows.size());
      ok(lp_ticket_tokens(inst, f.ticket, f.first.data(), static_cast<int32_t>(f.first.size())), "first tokens");
    }
    f.harvested = true;
    auto& queue = pending_[static_cast<size_t>(f.gpu)];
    const size_t idx = static_cast<size_t>(&f - log_.data());
    queue.erase(std::remove(queue.begin(), queue.end(), idx), queue.end());
  }

  // ---- timed window
  void open_window() {
    // Start from idle GPUs: the forwards queued before the window finish
    // outside it, on both clocks.
    for (Forward& f : log_) harvest(f);
    for (lp_instance* g : gpus_) ok(lp_timer_record(g, 0), "timer");
    win_.t0 = Clock::now();
  }
  void close_window() {
    for (lp_instance* g : gpus_) ok(lp_timer_record(g, 1), "timer");
    for (Forward& f : log_)
      if (f.in_window) harvest(f);  // every forward done, first tokens read on the host
    win_.wall_ms = ms_since(win_.t0);
    for (lp_instance* g : gpus_) {
      double ms = 0;
      ok(lp_timer_elapsed(g, 0, 1, &ms), "timer");
      win_.device_ms = std::max(win_.device_ms, ms);
    }
  }

  // ---- session residency
  std::int64_t kv_len(int g, std::int64_t sid) {
    int32_t np = 0;
    int64_t kv = 0;
    ok(lp_session_pages(gpus_[static_cast<size_t>(g)], sid, nullptr, 0, &np, &kv), "lp_session_pages");
    return kv;
  }

  void make_resident(int g, std::int64_t sid, Tokens H, bool inside) {
    if (H == 0) return;
    std::int64_t have = kv_len(g, sid);
    if (have >= H) return;
    // The copy holding the most positions elsewhere, if it beats ours.
    int best = -1;
    std::int64_t best_len = have;
    for (int h : holders_[sid]) {
      if (h == g) continue;
      const std::int64_t len = kv_len(h, sid);
      if (len > best_len) {
        best = h;
        best_len = len;
      }
    }
    if (best >= 0) {
      lp_instance* src = gpus_[static_cast<size_t>(best)];
      lp_instance* dst = gpus_[static_cast<size_t>(g)];
      if (chunking_on(sid) == best) {
        ok(lp_session_copy(src, dst, sid), "lp_session_copy");
      } else {
        ok(lp_session_migrate(src, dst, sid), "lp_session_migrate");
        holders_[sid].erase(best);
      }
      stats_.kv_migrations += 1;
      holders_[sid].insert(g);
      have = kv_len(g, sid);
      if (have >= H) return;
    }
    // Deterministic fill of the positions nobody has computed: [have, H).
    constexpr Tokens kFill = 2048;
    for (Tokens p = have; p < H; p += kFill) {
      const Tokens n = std::min(kFill, H - p);
      const lp_member m{-1, sid, n, p, 0, 0};
      std::vector<int32_t> toks;
      for (Tokens q = p; q < p + n; ++q) toks.push_back(lp_synth_token(seed_, sid, q, vocab_));
      const lp_shape shape{n, 1, LP_KIND_STANDARD};
      Forward f;
      f.gpu = g;
      f.fill = true;
      f.in_window = inside;
      f.tokens = n;
      submit(std::move(f), shape, &m, 1, toks.data());
      stats_.fill_forwards += 1;
      if (inside) win_.fills += 1;
    }
    holders_[sid].insert(g);
  }

  int chunking_on(std::int64_t sid) const {
    auto it = chunking_.find(sid);
    return it == chunking_.end() ? -1 : it->second;
  }

  void after_forward(int g, const ForwardCall& call) {
    for (const ForwardRow& row : call.rows) {
      const std::int64_t sid = row.session_id;
      auto& where = holders_[sid];
      where.insert(g);
      if (call.kind == ForwardKind::kLongChunk) {
        if (row.finishes_request) chunking_.erase(sid);
        else chunking_[sid] = g;
      }
      if (!row.finishes_request) continue;
      if (++turns_done_[sid] >= turns_[sid]) {  // the session's last turn in the stream: free every copy
        for (int h : where) ok(lp_session_release(gpus_[static_cast<size_t>(h)], sid), "lp_session_release");
        holders_.erase(sid);
        turns_done_.erase(sid);
        continue;
      }
      // Older copies elsewhere are stale now; drop them unless a long prompt
      // of this session is still chunking there.
      for (auto it = where.begin(); it != where.end();) {
        if (*it != g && chunking_on(sid) != *it) {
          ok(lp_session_release(gpus_[static_cast<size_t>(*it)], sid), "lp_session_release");
          it = where.erase(it);
        } else {
          ++it;
        }
      }
    }
  }

  static constexpr size_t kAhead = 12;  // forwards queued per GPU before results are collected

  std::vector<lp_instance*> gpus_;
  int32_t mode_;
  uint64_t seed_;
  int32_t vocab_;
  lp_sim_opts opts_;
  std::vector<std::vector<size_t>> pending_;  // per GPU: unharvested forwards (log_ indices, submit order)
  std::vector<std::int64_t> next_ticket_;      // per GPU: the ticket its next submit will get (known after one)
  std::vector<Forward> log_;
  std::int64_t dispatches_ = 0;
  std::unordered_map<std::int64_t, int> turns_, turns_done_;
  std::unordered_map<std::int64_t, std::set<int>> holders_;
  std::unordered_map<std::int64_t, int> chunking_;  // session -> GPU running its unfinished long prompt
  struct {
    std::int64_t gpu_forwards = 0, fill_forwards = 0, kv_migrations = 0, real_tokens = 0;
  } stats_;
  struct {
    std::int64_t dispatches = 0, requests = 0, fills = 0, kernels = 0, h2d = 0, d2h = 0;
    double device_ms = 0, wall_ms = 0;
    Clock::time_point t0;
  } win_;
};

// WALL mode without GPUs: every forward "runs" for its cost-model service
// time of real time, one at a time per lane (host-side tests of the wall
// clock: concurrency across lanes, arrival release, TTFT accounting).
class PacedBackend final : public ForwardBackend {
 public:
  std::uint64_t launch(const ForwardCall& call) override {
    due_.push_back({Clock::now() + std::chrono::duration_cast<Clock::duration>(
                                       std::chrono::duration<double, std::milli>(call.model_service_ms)),
                    call.model_service_ms});
    return due_.size();
  }
  double clock_ms(std::uint64_t, const ForwardCall& call) override { return call.model_service_ms; }
  bool poll(std::uint64_t h, double* ms) override {
    const auto& [when, svc] = due_[h - 1];
    if (Clock::now() < when) return false;
    *ms = svc;
    return true;
  }

 private:
  std::vector<std::pair<Clock::time_point, double>> due_;
};

ConfigMap config_from(const char* cfg_text, const char* overrides) {
  ConfigMap cfg = parse_config_text(cfg_text ? cfg_text : "");
  if (overrides && *overrides) apply_overrides(cfg, parse_config_text(overrides));
  return cfg;
}

struct RunOut {
  RunResult rr;
  std::unique_ptr<GpuTier> gpu;
};

RunOut run_mode(const Scenario& sc, int32_t mode, lp_instance** insts, int32_t n_insts, uint64_t token_seed,
                const lp_sim_opts& opts) {
  const std::vector<Request> reqs = build_workload(sc);
  RunOut out;
  if (mode == LP_SIM_COST_MODEL) {
    out.rr = run(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl);
    return out;
  }
  if (mode != LP_SIM_REPLAY && mode != LP_SIM_LIVE && mode != LP_SIM_WALL)
    throw ConfigError("unknown engine mode " + std::to_string(mode));
  const TierClock clock = mode == LP_SIM_WALL ? TierClock::kWall : TierClock::kVirtual;
  if (!insts || n_insts < 1) {
    if (mode != LP_SIM_WALL) throw ConfigError("REPLAY and LIVE modes need at least one GPU instance");
    PacedBackend paced;
    out.rr = run_tier(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl, paced, clock);
    return out;
  }
  if (opts.window_count > 0 && mode != LP_SIM_REPLAY) throw ConfigError("timed windows need REPLAY mode");
  lp_model_desc md{};
  ok(lp_instance_model(insts[0], &md), "lp_instance_model");
  out.gpu = std::make_unique<GpuTier>(insts, n_insts, mode, token_seed, md.vocab, reqs, opts);
  out.rr = run_tier(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl, *out.gpu, clock);
  return out;
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

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return LP_OK;
  } catch (const ShapeMismatch& e) {
    lp::set_last_error(e.what());
    return LP_ERR_SHAPE;
  } catch (const ConfigError& e) {
    lp::set_last_error(e.what());
    return LP_ERR_CONFIG;
  } catch (const InvalidConfig& e) {
    lp::set_last_error(e.what());
    return LP_ERR_CONFIG;
  } catch (const std::exception& e) {
    lp::set_last_error(e.what());
    return LP_ERR_INTERNAL;
  }
}

}  // namespace
}  // namespace laps

extern "C" {

int lp_sim_run_ex(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
                  lp_instance** insts, int32_t n_insts, uint64_t token_seed, const lp_sim_opts* opts,
                  lp_sim_stats* stats) {
  using namespace laps;
  return guarded([&] {
    const auto t0 = Clock::now();
    const lp_sim_opts o = opts ? *opts : lp_sim_opts{};
    RunOut run = run_mode(build_scenario(config_from(cfg_text, overrides)), mode, insts, n_insts, token_seed, o);
    const RunResult& rr = run.rr;
    if (out_dir && *out_dir) {
      std::filesystem::create_directories(out_dir);
      write_event_log(std::string(out_dir) + "/events.log", rr.log);
      write_metrics(std::string(out_dir) + "/metrics.json", rr.report);
      if (run.gpu) run.gpu->write(out_dir);
    }
    if (!stats) return;
    lp_sim_stats st{};
    if (run.gpu) run.gpu->fill_stats(st);
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
    st.engine_wall_s = ms_since(t0) / 1000.0;
    *stats = st;
  });
}

int lp_sim_run(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
               lp_instance** insts, int32_t n_insts, uint64_t token_seed, lp_sim_stats* stats) {
  return lp_sim_run_ex(cfg_text, overrides, out_dir, mode, insts, n_insts, token_seed, nullptr, stats);
}

int lp_sim_sweep(const char* cfg_text, const char* overrides, const char* out_dir, int32_t mode,
                 lp_instance** insts, int32_t n_insts, uint64_t token_seed, const char* param,
                 const char* values_csv) {
  using namespace laps;
  return guarded([&] {
    if (!param || !*param) throw ConfigError("sweep: empty parameter name");
    const ConfigMap base = config_from(cfg_text, overrides);
    std::vector<double> values;
    std::stringstream ss(values_csv ? values_csv : "");
    for (std::string item; std::getline(ss, item, ',');)
      if (!item.empty()) values.push_back(std::stod(item));
    if (values.empty()) throw ConfigError("sweep: --values parsed to an empty list");
    std::sort(values.begin(), values.end());
    static const char* kClassCols[] = {"completed",   "ttft_mean_ms", "ttft_p50_ms",  "ttft_p90_ms",
                                       "ttft_p99_ms", "rps",          "slo_violation", "mean_wait_ms",
                                       "batches",     "mean_depth",   "graph_hit_rate", "padding_overhead"};
    std::string csv = "param,value,arrivals,active_ms,migrations";
    for (const char* scope : {"overall_", "short_", "long_"})
      for (const char* col : kClassCols) csv += std::string(",") + scope + col;
    csv += '\n';
    for (double v : values) {
      ConfigMap cfg = base;  // fresh copy: scaling params read base values
      apply_sweep_param(cfg, param, v);
      const RunOut run = run_mode(build_scenario(cfg), mode, insts, n_insts, token_seed, lp_sim_opts{});
      const MetricsReport& m = run.rr.report;
      char head[160];
      std::snprintf(head, sizeof head, "%s,%.6f,%lld,%.6f,%lld", param, v, static_cast<long long>(m.arrivals),
                    m.active_ms, static_cast<long long>(m.migrations));
      std::string row = head;
      csv_class(row, m.overall);
      csv_class(row, m.short_cls);
      csv_class(row, m.long_cls);
      csv += row + '\n';
    }
    std::filesystem::create_directories(out_dir);
    std::ofstream os(std::string(out_dir) + "/sweep.csv", std::ios::binary);
    if (!os) throw std::runtime_error("sweep: cannot write sweep.csv");
    os << csv;
  });
}

int lp_sim_trace(const char* cfg_text, const char* overrides, const char* path) {
  using namespace laps;
  return guarded([&] {
    const auto reqs = build_workload(build_scenario(config_from(cfg_text, overrides)));
    FILE* f = std::fopen(path, "w");
    if (!f) throw ConfigError("cannot write trace dump");
    for (const auto& r : reqs) {
      std::fprintf(f, "%" PRId64 " %" PRId64 " %d %" PRId64 " %" PRId64 " %.17g ", r.id, r.session_id, r.turn,
                   r.new_tokens, r.history_tokens, r.arrival_ms);
      if (r.deadline_ms) std::fprintf(f, "%.17g\n", *r.deadline_ms);
      else std::fprintf(f, "none\n");
    }
    std::fclose(f);
  });
}

}  // extern "C"
