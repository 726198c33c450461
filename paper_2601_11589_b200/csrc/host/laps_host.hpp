// Host engine of the LAPS prefill tier — the reference's scheduler API kept
// unchanged (same type names, fields, defaults and function signatures as
// /root/reference/proj/include/prefillsim/*.hpp), re-implemented for this
// framework. The one structural change: the three forward call sites
// (sim.cpp:254, :283, :357) go through `ForwardBackend`, so the same engine
// runs against the closed-form cost model (replay / parity) or a B200
// prefill instance (live, measured service times).
//
// `namespace prefillsim` is an alias of `laps`, so reference callers compile
// against this header unchanged.
#pragma once

#include <cstdint>
#include <deque>
#include <limits>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace laps {

// ---------------------------------------------------------------- types.hpp
using Tokens = std::int64_t;     // all sizes in tokens
using RequestId = std::int64_t;  // all times in ms

// ----------------------------------------------------------- cost_model.hpp
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct CostParams {  // cost_model.hpp:24-29
  double alpha = 2e-5;
  double beta = 0.005;
  double gamma_w = 0.01012;
  double gamma_r = 0.002;
};
struct ExecOverheads {  // cost_model.hpp:32-36
  double kappa_graph_ms = 0.05;
  double kappa_std_ms = 0.5;
  double eta = 0.7;
};
struct RooflineParams {
  double p_peak = 1e15;
  double b_mem = 4e12;
  double bytes_per_token = 131072.0;
  double ops_per_token = 128000.0;
};
enum class ShapeKind { kGraph, kStandard };
struct BatchShape {  // cost_model.hpp:60-64
  Tokens l_pad = 0;
  int depth = 0;
  ShapeKind kind = ShapeKind::kStandard;
};
struct LatencyTerms {
  double comp_ms = 0;
  double mem_ms = 0;
  double total_ms() const { return comp_ms + mem_ms; }
};
using MemberShape = std::pair<Tokens, Tokens>;  // (L, H)

void validate(const CostParams& p);
void validate(const ExecOverheads& o);
void validate(const RooflineParams& r);
LatencyTerms compute_latency(double new_tokens, double history_tokens, const CostParams& p);
double prefill_boundary(const CostParams& p);
double reprefill_boundary(const CostParams& p, double history_tokens);
double batch_service_time(const BatchShape& shape, std::span<const MemberShape> members,
                          const CostParams& p, const ExecOverheads& o);
double packed_service_time(std::span<const MemberShape> members, const CostParams& p,
                           const ExecOverheads& o);

// ------------------------------------------------------------- workload.hpp
struct Request {  // workload.hpp:17-27
  RequestId id = 0;
  std::int64_t session_id = 0;
  int turn = 1;
  Tokens new_tokens = 1;
  Tokens history_tokens = 0;
  double arrival_ms = 0;
  std::optional<double> deadline_ms;
  bool operator==(const Request&) const = default;
};
struct LengthDist {
  Tokens lo = 1;
  Tokens hi = 1;
};
struct IntRange {
  int lo = 1;
  int hi = 1;
};
struct SynthConfig {  // workload.hpp:40-50
  double lambda_per_ms = 0.01;
  double short_fraction = 0.63;
  double short_fraction_later = 0.63;
  LengthDist short_len{8, 255};
  LengthDist long_len{256, 2048};
  IntRange turns_per_session{1, 1};
  std::optional<double> slo_offset_ms;
  std::optional<double> duration_ms;
  std::uint64_t seed = 1;
};
struct InvalidConfig : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  ParseError(const std::string& msg, int line)
      : std::runtime_error("line " + std::to_string(line) + ": " + msg), line_number(line) {}
  int line_number;
};
struct InvariantViolation : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::vector<Request> synth_stream(const SynthConfig& cfg, double duration_ms);
std::vector<Request> load_trace(const std::string& path);
void save_trace(const std::string& path, std::span<const Request> requests);
enum class LengthClass { kShort, kLong };
LengthClass classify(const Request& r, Tokens l_m_first, Tokens l_m_re);
std::vector<Request> merge_streams(std::vector<Request> a, std::vector<Request> b);
std::vector<Request> shift_stream(std::vector<Request> v, double dt_ms);

// ------------------------------------------------------------ scheduler.hpp
struct GraphGrid {  // scheduler.hpp:21-32
  std::vector<Tokens> lengths{8, 16, 32, 64, 128, 256};
  std::vector<int> depths{1, 2, 4, 8, 16, 32, 64};
  double mem_per_graph_bytes = 240.0 * 1024 * 1024;
  double mem_budget_bytes = 16.0 * 1024 * 1024 * 1024;
  Tokens max_length() const { return lengths.back(); }
  int max_depth() const { return depths.back(); }
  bool graphs_enabled() const { return mem_per_graph_bytes <= mem_budget_bytes; }
};
void validate(const GraphGrid& g);

enum class SchedMode { kSla, kDeadlineFree };
struct SchedConfig {  // scheduler.hpp:38-52
  double w_min_ms = 1.0;
  double w_max_ms = 50.0;
  double sigma_ms = 10.0;
  double delta_ms = 5.0;
  double t_max_ms = 100.0;
  double epsilon_per_ms = 1e-6;
  Tokens m_s_tokens = 2048;
  Tokens c_l_tokens = 512;
  SchedMode mode = SchedMode::kSla;
  Tokens l_m_first = 256;
  Tokens l_m_re = 256;
  double s_hat_init_ms = 1.0;
  double ewma_decay = 0.2;
};
void validate(const SchedConfig& c);

struct AwdState {  // scheduler.hpp:61-72
  double w = 0;
  int d = 1;
  double s_hat = 0;
  double r_hat = 0;
  bool round_open = false;
  double round_start = 0;
  int arrivals_in_round = 0;
  std::uint64_t round_id = 0;
  double next_check = 0;
};
AwdState make_awd_state(const SchedConfig& cfg, const GraphGrid& grid);

enum class DispatchReason { kDepthReached, kWindowExpired, kSlaBreak, kHolCap, kTokenMax };
const char* to_string(DispatchReason r);

struct BatchPlan {  // scheduler.hpp:87-93
  std::vector<RequestId> members;
  BatchShape shape;
  double dispatch_ms = 0;
  DispatchReason reason = DispatchReason::kDepthReached;
  Tokens real_tokens = 0;
};

std::optional<Tokens> bucket_of(Tokens new_tokens, const GraphGrid& grid);
std::optional<BatchShape> nearest_graph(std::span<const Tokens> lengths, const GraphGrid& grid);
std::vector<size_t> group_candidates(const std::deque<Request>& queue, const GraphGrid& grid, int cap);
double sla_window(const std::deque<Request>& queue, double now, const AwdState& st, const SchedConfig& cfg);
double graph_window(const AwdState& st, int current_depth, const SchedConfig& cfg);
double combined_window(const std::deque<Request>& queue, double now, int current_depth,
                       const AwdState& st, const SchedConfig& cfg);
double clip_window(double w, const SchedConfig& cfg);
void awd_update_after_dispatch(AwdState& st, int depth, double tau_fill, const SchedConfig& cfg);
void observe_service(AwdState& st, double service_ms, int depth, const SchedConfig& cfg);

struct AwdDecision {
  std::optional<BatchPlan> plan;
  double next_check_ms = 0;
};
AwdDecision awd_step(AwdState& st, const std::deque<Request>& queue, double now, const GraphGrid& grid,
                     const SchedConfig& cfg);
AwdDecision token_max_admit(AwdState& st, const std::deque<Request>& queue, double now,
                            const GraphGrid& grid, const SchedConfig& cfg);

struct ChunkDesc {
  int index = 0;
  Tokens tokens = 0;
  Tokens history = 0;
};
std::vector<ChunkDesc> long_chunk_dispatch(const Request& r, const SchedConfig& cfg);

// ----------------------------------------------------------- controller.hpp
struct InstanceStats {
  double q = 0;
  double e = 0;
  double u = 0;
};
struct ControllerConfig {  // controller.hpp:20-29
  double dt_ms = 100;
  double t_cool_ms = 500;
  double tau_hyst = 0.25;
  int n_min = 1;
  double w_q = 1.0;
  double w_e = 10.0;
  double w_u = 5.0;
  int aggregator_percentile = 90;
};
enum class PoolKind { kShort, kLong };
struct PoolState {
  std::vector<PoolKind> assignment;
  double t_last_ms = -std::numeric_limits<double>::infinity();
  int n_short() const;
  int n_long() const;
};
enum class MigrationDir { kLongToShort, kShortToLong };
const char* to_string(MigrationDir d);
struct EmptyPool : std::runtime_error {
  EmptyPool() : std::runtime_error("pool has no instances to aggregate") {}
};
void validate(const ControllerConfig& cfg, int n_instances);
double pressure(const InstanceStats& s, const ControllerConfig& cfg);
double aggregate(std::span<const double> scores, int percentile);
std::optional<MigrationDir> decide(double p_s, double p_l, PoolState& state, const ControllerConfig& cfg,
                                   double now_ms);

// ------------------------------------------------------------ event_log.hpp
enum class EventKind { kArrival, kDispatch, kBatchComplete, kControllerTick, kMigration };
const char* to_string(EventKind k);
struct LogRecord {  // event_log.hpp:25-58
  double t = 0;
  std::int64_t seq = 0;
  EventKind kind = EventKind::kArrival;
  RequestId req = -1;
  Tokens length = 0;
  Tokens history = 0;
  std::optional<double> deadline_ms;
  int inst = -1;
  std::vector<RequestId> reqs;
  std::string cls;
  std::string reason;
  Tokens l_pad = 0;
  int depth = 0;
  bool graph = false;
  Tokens real_tokens = 0;
  Tokens padded_tokens = 0;
  int chunk = 0;
  int chunks_total = 0;
  double service_ms = 0;
  bool final_chunk = true;
  int n_short = 0;
  int n_long = 0;
  double p_short = 0;
  double p_long = 0;
  bool migrated = false;
  std::string direction;
};
std::string serialize(const LogRecord& r);
void write_event_log(const std::string& path, std::span<const LogRecord> log);

// -------------------------------------------------------------- metrics.hpp
struct EmptySamples : std::runtime_error {
  EmptySamples() : std::runtime_error("no samples") {}
};
double percentile(std::span<const double> samples, double q);
double slo_violation_rate(std::span<const double> ttfts_ms, double slo_ms);
struct ClassMetrics {
  std::int64_t completed = 0;
  double ttft_mean_ms = 0;
  double ttft_p50_ms = 0;
  double ttft_p90_ms = 0;
  double ttft_p99_ms = 0;
  double rps = 0;
  double slo_violation = 0;
  double mean_wait_ms = 0;
  std::int64_t batches = 0;
  double mean_depth = 0;
  double graph_hit_rate = 0;
  double padding_overhead = 0;
};
struct MetricsReport {
  double slo_ms = 400;
  double active_ms = 0;
  std::int64_t arrivals = 0;
  std::int64_t migrations = 0;
  ClassMetrics overall;
  ClassMetrics short_cls;
  ClassMetrics long_cls;
};
MetricsReport metrics_from_log(std::span<const LogRecord> log, double slo_ms);
std::string to_json(const MetricsReport& m);
void write_metrics(const std::string& path, const MetricsReport& m);

// ------------------------------------------------------------------ sim.hpp
enum class Policy { kLaps, kFcfsUnified, kBucketNoDisagg };
enum class Disagg { kTemporal, kSpatial };
Policy parse_policy(const std::string& s);
Disagg parse_disagg(const std::string& s);
const char* to_string(Policy p);
const char* to_string(Disagg d);

struct SimConfig {  // sim.hpp:24-36
  int n_instances = 1;
  Policy policy = Policy::kLaps;
  Disagg disagg = Disagg::kTemporal;
  bool controller_on = false;
  std::uint64_t seed = 1;
  double duration_ms = 10000;
  double slo_ms = 400;
  int initial_short_instances = -1;
  Tokens unified_token_budget = 8192;
  int unified_max_batch = 64;
  double startup_delay_ms = 0;
};
void validate(const SimConfig& c);

struct RunResult {
  std::vector<LogRecord> log;
  MetricsReport report;
};

// ---- the forward boundary (NEW; replaces the three cost-model call sites)
// One dispatched batch as the engine hands it to a backend.
struct ForwardRow {
  RequestId req_id = 0;
  std::int64_t session_id = 0;
  Tokens new_tokens = 0;  // L (chunk length for long chunks)
  Tokens history = 0;     // H (+ preceding chunk tokens)
  bool finishes_request = true;
};
enum class ForwardKind { kAwdBatch, kLongChunk, kPacked };
struct ForwardCall {
  int inst = 0;
  double now_ms = 0;
  ForwardKind kind = ForwardKind::kAwdBatch;
  BatchShape shape;                 // kPacked: l_pad = max L, depth = count
  std::vector<ForwardRow> rows;     // real members in plan order (no dummy rows)
  double model_service_ms = 0;      // what the reference cost model says
};

// How the engine's clock advances.
//   kVirtual  discrete-event time: a forward completes clock_ms() after it
//             was launched (the reference semantics; byte-identical logs).
//   kWall     steady_clock time: arrivals are released in real time and a
//             forward completes when poll() says so; lanes run concurrently.
enum class TierClock { kVirtual, kWall };

// Where dispatched forwards go. launch() must not block on the forward
// itself, so several lanes (GPUs) overlap; a handle of 0 means "nothing to
// wait for" (closed form).
class ForwardBackend {
 public:
  virtual ~ForwardBackend() = default;
  virtual std::uint64_t launch(const ForwardCall& call) = 0;
  // Virtual clock: the service time the clock advances by (may block when it
  // has to be measured).
  virtual double clock_ms(std::uint64_t handle, const ForwardCall& call) = 0;
  // Wall clock: true once the forward finished; *service_ms = its duration.
  virtual bool poll(std::uint64_t handle, double* service_ms) = 0;
  // The run is over: drain whatever is still queued.
  virtual void finish_run() {}
};
// The reference semantics: service time = closed-form cost model.
class CostModelBackend final : public ForwardBackend {
 public:
  std::uint64_t launch(const ForwardCall&) override { return 0; }
  double clock_ms(std::uint64_t, const ForwardCall& call) override { return call.model_service_ms; }
  bool poll(std::uint64_t, double*) override {
    throw std::logic_error("the closed-form backend has no wall-clock completions");
  }
};

RunResult run(const SimConfig& sim, const std::vector<Request>& requests, const CostParams& cost,
              const ExecOverheads& overheads, const SchedConfig& sched, const GraphGrid& grid,
              const ControllerConfig& ctrl);
RunResult run_with_backend(const SimConfig& sim, const std::vector<Request>& requests,
                           const CostParams& cost, const ExecOverheads& overheads,
                           const SchedConfig& sched, const GraphGrid& grid,
                           const ControllerConfig& ctrl, ForwardBackend& backend);
RunResult run_tier(const SimConfig& sim, const std::vector<Request>& requests, const CostParams& cost,
                   const ExecOverheads& overheads, const SchedConfig& sched, const GraphGrid& grid,
                   const ControllerConfig& ctrl, ForwardBackend& backend, TierClock clock);

// --------------------------------------------------------------- config.hpp
using ConfigMap = std::map<std::string, std::string>;
ConfigMap parse_config_text(const std::string& text);
ConfigMap parse_config_file(const std::string& path);
void apply_overrides(ConfigMap& base, const ConfigMap& overrides);
struct Scenario {
  SimConfig sim;
  CostParams cost;
  ExecOverheads overheads;
  RooflineParams roofline;
  SchedConfig sched;
  GraphGrid grid;
  ControllerConfig ctrl;
  SynthConfig workload;
  std::optional<SynthConfig> workload2;
  double workload2_shift_ms = 0;
  std::optional<std::string> trace_path;
};
Scenario build_scenario(const ConfigMap& cfg);
std::vector<Request> build_workload(const Scenario& sc);
void apply_sweep_param(ConfigMap& cfg, const std::string& param, double value);
RunResult run_scenario(const Scenario& sc);

}  // namespace laps

namespace prefillsim = laps;
