// Closed-form pieces of the host engine: the analytical service-time model
// (the forward stand-in, cost_model.cpp:36-61, 128-158) and the Alg. 2
// controller arithmetic (controller.cpp:9-65). Expression order follows the
// reference term by term so double results are bit-identical.
#include <algorithm>
#include <cmath>

#include "laps_host.hpp"

namespace laps {

void validate(const CostParams& p) {
  if (!(p.alpha > 0) || !std::isfinite(p.alpha)) throw ConfigError("cost.alpha must be finite and > 0");
  for (double v : {p.beta, p.gamma_w, p.gamma_r})
    if (v < 0 || !std::isfinite(v)) throw ConfigError("cost coefficients must be finite and >= 0");
}

void validate(const ExecOverheads& o) {
  if (!(o.eta > 0) || o.eta > 1.0) throw ConfigError("cost.eta must be in (0,1]");
  if (o.kappa_graph_ms < 0 || o.kappa_std_ms < o.kappa_graph_ms)
    throw ConfigError("need 0 <= kappa_graph <= kappa_std");
}

void validate(const RooflineParams& r) {
  for (double v : {r.p_peak, r.b_mem, r.bytes_per_token, r.ops_per_token})
    if (!(v > 0) || !std::isfinite(v)) throw ConfigError("roofline parameters must be finite and > 0");
}

LatencyTerms compute_latency(double L, double H, const CostParams& p) {
  // t_comp = alpha*L*(L+2H) + beta*L ; t_mem = gamma_w*L + gamma_r*H
  return LatencyTerms{p.alpha * L * (L + 2.0 * H) + p.beta * L, p.gamma_w * L + p.gamma_r * H};
}

double prefill_boundary(const CostParams& p) { return std::max(0.0, (p.gamma_w - p.beta) / p.alpha); }

double reprefill_boundary(const CostParams& p, double H) {
  // Nonnegative root of alpha*L^2 + b*L - gamma_r*H with b = 2*alpha*H + beta - gamma_w;
  // the rationalised form is used when b >= 0 to avoid cancellation.
  const double b = 2.0 * p.alpha * H + p.beta - p.gamma_w;
  const double sq = std::sqrt(b * b + 4.0 * p.alpha * p.gamma_r * H);
  const double root = b >= 0 ? ((b + sq) > 0 ? 2.0 * p.gamma_r * H / (b + sq) : 0.0)
                             : (-b + sq) / (2.0 * p.alpha);
  return std::max(0.0, root);
}

double batch_service_time(const BatchShape& shape, std::span<const MemberShape> members,
                          const CostParams& p, const ExecOverheads& o) {
  if (static_cast<int>(members.size()) != shape.depth) {
    throw ShapeMismatch("member count " + std::to_string(members.size()) + " != shape depth " +
                        std::to_string(shape.depth));
  }
  double acc = 0;
  for (const auto& m : members) {
    if (m.first > shape.l_pad) {
      throw ShapeMismatch("member length " + std::to_string(m.first) + " exceeds l_pad " +
                          std::to_string(shape.l_pad));
    }
    // Padding is billed in full: every row costs a full l_pad row.
    acc += compute_latency(static_cast<double>(shape.l_pad), static_cast<double>(m.second), p).total_ms();
  }
  const double kappa = shape.kind == ShapeKind::kGraph ? o.kappa_graph_ms : o.kappa_std_ms;
  return kappa + std::pow(static_cast<double>(shape.depth), o.eta - 1.0) * acc;
}

double packed_service_time(std::span<const MemberShape> members, const CostParams& p,
                           const ExecOverheads& o) {
  double acc = 0;
  for (const auto& m : members)
    acc += compute_latency(static_cast<double>(m.first), static_cast<double>(m.second), p).total_ms();
  return o.kappa_std_ms + acc;
}

// ------------------------------------------------------------- controller
int PoolState::n_short() const {
  return static_cast<int>(std::count(assignment.begin(), assignment.end(), PoolKind::kShort));
}
int PoolState::n_long() const { return static_cast<int>(assignment.size()) - n_short(); }

const char* to_string(MigrationDir d) {
  return d == MigrationDir::kLongToShort ? "long_to_short" : "short_to_long";
}

void validate(const ControllerConfig& cfg, int n_instances) {
  if (!(cfg.dt_ms > 0)) throw ConfigError("control period must be > 0");
  if (cfg.t_cool_ms < 0) throw ConfigError("cool-down must be >= 0");
  if (cfg.tau_hyst < 0) throw ConfigError("hysteresis must be >= 0");
  if (cfg.n_min < 0) throw ConfigError("n_min must be >= 0");
  if (2 * cfg.n_min > n_instances) throw ConfigError("n_min * 2 exceeds the instance count");
  for (double w : {cfg.w_q, cfg.w_e, cfg.w_u})
    if (w < 0) throw ConfigError("pressure weights must be >= 0");
  if (cfg.aggregator_percentile < 1 || cfg.aggregator_percentile > 100)
    throw ConfigError("aggregator percentile must be in [1, 100]");
}

double pressure(const InstanceStats& s, const ControllerConfig& cfg) {
  return cfg.w_q * s.q + cfg.w_e * s.e - cfg.w_u * s.u;
}

double aggregate(std::span<const double> scores, int pct) {
  if (scores.empty()) throw EmptyPool();
  std::vector<double> v(scores.begin(), scores.end());
  std::sort(v.begin(), v.end());
  // nearest rank ceil(p*n/100) in integer arithmetic
  const size_t n = v.size();
  const size_t rank = std::clamp<size_t>((static_cast<size_t>(pct) * n + 99) / 100, 1, n);
  return v[rank - 1];
}

std::optional<MigrationDir> decide(double p_s, double p_l, PoolState& st, const ControllerConfig& cfg,
                                   double now) {
  if (now - st.t_last_ms < cfg.t_cool_ms) return std::nullopt;
  const double gain = 1.0 + cfg.tau_hyst;
  std::optional<MigrationDir> dir;
  if (p_s > gain * p_l && st.n_long() > cfg.n_min) {
    dir = MigrationDir::kLongToShort;
  } else if (p_l > gain * p_s && st.n_short() > cfg.n_min) {
    dir = MigrationDir::kShortToLong;
  }
  if (dir) st.t_last_ms = now;
  return dir;
}

}  // namespace laps
