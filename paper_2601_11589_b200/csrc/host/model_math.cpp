// Closed-form parts of the host engine.
//
//  * The Alg. 2 pool controller's arithmetic (reference controller.cpp:9-65):
//    per-instance pressure, the percentile aggregate of a pool, the
//    hysteresis / cool-down / minimum-pool decision.
//  * The analytical service-time model the reference uses in place of a
//    forward (cost_model.cpp:36-61, 128-158). It still drives the REPLAY
//    clock (so batch composition matches the reference) and the cost-model
//    mode; on the GPU path the real forward replaces it. The floating-point
//    expressions are the reference's term for term (the clock must be
//    bit-identical), the surrounding code is this repo's own.
#include <algorithm>
#include <cmath>

#include "laps_host.hpp"

namespace laps {

namespace {

struct Rule {
  bool broken;
  const char* why;
};
void enforce(std::initializer_list<Rule> rules) {
  for (const Rule& r : rules)
    if (r.broken) throw ConfigError(r.why);
}

bool finite_positive(double v) { return v > 0 && std::isfinite(v); }
bool finite_nonnegative(double v) { return v >= 0 && std::isfinite(v); }

}  // namespace

// ---------------------------------------------------------------- controller
int PoolState::n_long() const {
  int n = 0;
  for (PoolKind k : assignment) n += k == PoolKind::kLong ? 1 : 0;
  return n;
}
int PoolState::n_short() const { return static_cast<int>(assignment.size()) - n_long(); }

const char* to_string(MigrationDir d) {
  switch (d) {
    case MigrationDir::kShortToLong: return "short_to_long";
    case MigrationDir::kLongToShort: return "long_to_short";
  }
  return "?";
}

void validate(const ControllerConfig& c, int n_instances) {
  enforce({
      {!(c.dt_ms > 0), "ctrl.dt_ms must be > 0"},
      {c.t_cool_ms < 0, "ctrl.t_cool_ms must be >= 0"},
      {c.tau_hyst < 0, "ctrl.tau_hyst must be >= 0"},
      {c.n_min < 0, "ctrl.n_min must be >= 0"},
      {c.n_min * 2 > n_instances, "ctrl.n_min leaves no room for two pools of that size"},
      {c.w_q < 0 || c.w_e < 0 || c.w_u < 0, "ctrl weights w_q, w_e, w_u must be >= 0"},
      {c.aggregator_percentile < 1 || c.aggregator_percentile > 100, "ctrl percentile must be in 1..100"},
  });
}

// Queue pressure plus lateness, minus how busy the instance already is.
double pressure(const InstanceStats& s, const ControllerConfig& c) {
  return c.w_q * s.q + c.w_e * s.e - c.w_u * s.u;
}

// Pool score: the nearest-rank p-th percentile of its instances' pressures,
// rank ceil(p n / 100) computed in integers.
double aggregate(std::span<const double> scores, int pct) {
  if (scores.empty()) throw EmptyPool();
  const size_t n = scores.size();
  size_t rank = (static_cast<size_t>(pct) * n + 99) / 100;
  rank = std::min(std::max<size_t>(rank, 1), n);
  std::vector<double> v(scores.begin(), scores.end());
  std::nth_element(v.begin(), v.begin() + static_cast<long>(rank - 1), v.end());
  return v[rank - 1];
}

// Move one instance toward the pool under more pressure, when it is ahead
// by the hysteresis margin, the donor pool keeps n_min instances, and the
// last move is at least t_cool ago.
std::optional<MigrationDir> decide(double p_s, double p_l, PoolState& pools, const ControllerConfig& c,
                                   double now) {
  if (now - pools.t_last_ms < c.t_cool_ms) return std::nullopt;
  const double margin = 1.0 + c.tau_hyst;
  const bool short_starved = p_s > margin * p_l && pools.n_long() > c.n_min;
  const bool long_starved = !short_starved && p_l > margin * p_s && pools.n_short() > c.n_min;
  if (!short_starved && !long_starved) return std::nullopt;
  pools.t_last_ms = now;
  return short_starved ? MigrationDir::kLongToShort : MigrationDir::kShortToLong;
}

// ---------------------------------------------------------------- cost model
void validate(const RooflineParams& r) {
  enforce({{!finite_positive(r.p_peak) || !finite_positive(r.b_mem) || !finite_positive(r.bytes_per_token) ||
                !finite_positive(r.ops_per_token),
            "roofline parameters must be finite and > 0"}});
}

void validate(const ExecOverheads& o) {
  enforce({
      {!(o.eta > 0) || o.eta > 1.0, "exec.eta must lie in (0, 1]"},
      {o.kappa_graph_ms < 0 || o.kappa_std_ms < o.kappa_graph_ms, "exec: need 0 <= kappa_graph <= kappa_std"},
  });
}

void validate(const CostParams& p) {
  enforce({
      {!finite_positive(p.alpha), "cost.alpha must be finite and > 0"},
      {!finite_nonnegative(p.beta) || !finite_nonnegative(p.gamma_w) || !finite_nonnegative(p.gamma_r),
       "cost.beta, cost.gamma_w, cost.gamma_r must be finite and >= 0"},
  });
}

// One row of L new tokens over H cached ones: compute (quadratic attention
// + linear projections) and memory (KV write + KV read) terms.
LatencyTerms compute_latency(double L, double H, const CostParams& p) {
  LatencyTerms t;
  t.comp_ms = p.alpha * L * (L + 2.0 * H) + p.beta * L;
  t.mem_ms = p.gamma_w * L + p.gamma_r * H;
  return t;
}

// L at which a fresh prompt's compute time overtakes its memory time.
double prefill_boundary(const CostParams& p) {
  const double crossing = (p.gamma_w - p.beta) / p.alpha;
  return crossing > 0.0 ? crossing : 0.0;
}

// Same crossing for a re-prefill over H cached tokens: the nonnegative root
// of alpha L^2 + b L - gamma_r H = 0, b = 2 alpha H + beta - gamma_w, in the
// cancellation-free form when b >= 0.
double reprefill_boundary(const CostParams& p, double H) {
  const double b = 2.0 * p.alpha * H + p.beta - p.gamma_w;
  const double disc = std::sqrt(b * b + 4.0 * p.alpha * p.gamma_r * H);
  double L = 0.0;
  if (b < 0) L = (-b + disc) / (2.0 * p.alpha);
  else if (b + disc > 0) L = 2.0 * p.gamma_r * H / (b + disc);
  return L > 0.0 ? L : 0.0;
}

// A padded batch: every row is billed as a full l_pad row (dummy rows up to
// the depth too), the sum scaled by depth^(eta - 1), plus the launch cost of
// a graph replay or an eager launch.
double batch_service_time(const BatchShape& shape, std::span<const MemberShape> members, const CostParams& p,
                          const ExecOverheads& o) {
  if (members.size() != static_cast<size_t>(std::max(shape.depth, 0)) || shape.depth < 0)
    throw ShapeMismatch("batch of " + std::to_string(members.size()) + " rows for a graph of depth " +
                        std::to_string(shape.depth));
  const double row_len = static_cast<double>(shape.l_pad);
  double rows_ms = 0;
  for (const MemberShape& m : members) {
    if (m.first > shape.l_pad)
      throw ShapeMismatch("row of " + std::to_string(m.first) + " tokens does not fit l_pad " +
                          std::to_string(shape.l_pad));
    rows_ms += compute_latency(row_len, static_cast<double>(m.second), p).total_ms();
  }
  const double launch = shape.kind == ShapeKind::kGraph ? o.kappa_graph_ms : o.kappa_std_ms;
  const double batching = std::pow(static_cast<double>(shape.depth), o.eta - 1.0);
  return launch + batching * rows_ms;
}

// The FCFS baseline's packed batch: no padding, no batching discount.
double packed_service_time(std::span<const MemberShape> members, const CostParams& p, const ExecOverheads& o) {
  double rows_ms = 0;
  for (const MemberShape& m : members)
    rows_ms += compute_latency(static_cast<double>(m.first), static_cast<double>(m.second), p).total_ms();
  return o.kappa_std_ms + rows_ms;
}

}  // namespace laps
