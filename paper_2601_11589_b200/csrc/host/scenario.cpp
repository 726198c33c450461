// Flat dotted-key configuration (`section.key = value`, '#' comments, unknown
// or duplicate keys rejected) with the reference's key names and defaults
// (config.cpp:116-372), scenario assembly and workload construction.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>

#include "laps_host.hpp"

namespace laps {

namespace {

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
  while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
  return s.substr(a, b - a);
}

template <typename T, typename F>
T parse_full(const std::string& key, const std::string& v, F fn, const char* what) {
  size_t pos = 0;
  T out{};
  try {
    out = fn(v, &pos);
  } catch (const std::exception&) {
    throw ConfigError(key + ": not " + what + ": '" + v + "'");
  }
  if (pos != v.size()) throw ConfigError(key + ": trailing junk in " + what + ": '" + v + "'");
  return out;
}

double num(const std::string& k, const std::string& v) {
  return parse_full<double>(k, v, [](const std::string& s, size_t* p) { return std::stod(s, p); }, "a number");
}
std::int64_t integer(const std::string& k, const std::string& v) {
  return parse_full<std::int64_t>(k, v, [](const std::string& s, size_t* p) { return std::stoll(s, p); },
                                  "an integer");
}
std::uint64_t uinteger(const std::string& k, const std::string& v) {
  return parse_full<std::uint64_t>(k, v, [](const std::string& s, size_t* p) { return std::stoull(s, p); },
                                   "an unsigned integer");
}
bool boolean(const std::string& k, const std::string& v) {
  if (v == "1" || v == "true" || v == "on" || v == "yes") return true;
  if (v == "0" || v == "false" || v == "off" || v == "no") return false;
  throw ConfigError(k + ": not a boolean: '" + v + "'");
}
template <typename T>
std::vector<T> int_list(const std::string& k, const std::string& v) {
  std::vector<T> out;
  std::stringstream ss(v);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(static_cast<T>(integer(k, trim(item))));
  if (out.empty()) throw ConfigError(k + ": empty list");
  return out;
}

using Setter = std::function<void(const std::string& key, const std::string& v)>;

bool set_synth(SynthConfig& w, const std::string& sub, const std::string& k, const std::string& v) {
  const std::map<std::string, Setter> table = {
      {"lambda_per_ms", [&](auto& key, auto& val) { w.lambda_per_ms = num(key, val); }},
      {"short_fraction", [&](auto& key, auto& val) { w.short_fraction = num(key, val); }},
      {"short_fraction_later", [&](auto& key, auto& val) { w.short_fraction_later = num(key, val); }},
      {"short_lo", [&](auto& key, auto& val) { w.short_len.lo = integer(key, val); }},
      {"short_hi", [&](auto& key, auto& val) { w.short_len.hi = integer(key, val); }},
      {"long_lo", [&](auto& key, auto& val) { w.long_len.lo = integer(key, val); }},
      {"long_hi", [&](auto& key, auto& val) { w.long_len.hi = integer(key, val); }},
      {"turns_lo", [&](auto& key, auto& val) { w.turns_per_session.lo = static_cast<int>(integer(key, val)); }},
      {"turns_hi", [&](auto& key, auto& val) { w.turns_per_session.hi = static_cast<int>(integer(key, val)); }},
      {"slo_offset_ms", [&](auto& key, auto& val) { w.slo_offset_ms = num(key, val); }},
      {"duration_ms", [&](auto& key, auto& val) { w.duration_ms = num(key, val); }},
      {"seed", [&](auto& key, auto& val) { w.seed = uinteger(key, val); }},
  };
  auto it = table.find(sub);
  if (it == table.end()) return false;
  it->second(k, v);
  return true;
}

}  // namespace

ConfigMap parse_config_text(const std::string& text) {
  ConfigMap out;
  std::istringstream in(text);
  std::string line;
  for (int n = 1; std::getline(in, line); ++n) {
    if (const size_t h = line.find('#'); h != std::string::npos) line.resize(h);
    line = trim(line);
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError("config line " + std::to_string(n) + ": expected key=value");
    const std::string key = trim(line.substr(0, eq));
    if (key.empty()) throw ConfigError("config line " + std::to_string(n) + ": empty key");
    if (out.count(key)) throw ConfigError("config line " + std::to_string(n) + ": duplicate key '" + key + "'");
    out[key] = trim(line.substr(eq + 1));
  }
  return out;
}

ConfigMap parse_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot read config file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_config_text(ss.str());
}

void apply_overrides(ConfigMap& base, const ConfigMap& overrides) {
  for (const auto& [k, v] : overrides) base[k] = v;
}

Scenario build_scenario(const ConfigMap& cfg) {
  Scenario sc;
  // The model preset sets the per-graph footprint before explicit grid keys.
  if (auto it = cfg.find("grid.model_preset"); it != cfg.end()) {
    static const std::map<std::string, double> mib = {{"7b", 228.0}, {"14b", 240.0}, {"32b", 277.0}};
    auto p = mib.find(it->second);
    if (p == mib.end())
      throw ConfigError("grid.model_preset: unknown preset '" + it->second + "' (expected 7b, 14b, or 32b)");
    sc.grid.mem_per_graph_bytes = p->second * 1024 * 1024;
  }
  const std::map<std::string, Setter> keys = {
      {"sim.instances", [&](auto& k, auto& v) { sc.sim.n_instances = static_cast<int>(integer(k, v)); }},
      {"sim.policy", [&](auto&, auto& v) { sc.sim.policy = parse_policy(v); }},
      {"sim.disagg", [&](auto&, auto& v) { sc.sim.disagg = parse_disagg(v); }},
      {"sim.controller", [&](auto& k, auto& v) { sc.sim.controller_on = boolean(k, v); }},
      {"sim.seed", [&](auto& k, auto& v) { sc.sim.seed = uinteger(k, v); }},
      {"sim.duration_ms", [&](auto& k, auto& v) { sc.sim.duration_ms = num(k, v); }},
      {"sim.slo_ms", [&](auto& k, auto& v) { sc.sim.slo_ms = num(k, v); }},
      {"sim.initial_short_instances",
       [&](auto& k, auto& v) { sc.sim.initial_short_instances = static_cast<int>(integer(k, v)); }},
      {"sim.token_budget", [&](auto& k, auto& v) { sc.sim.unified_token_budget = integer(k, v); }},
      {"sim.max_batch", [&](auto& k, auto& v) { sc.sim.unified_max_batch = static_cast<int>(integer(k, v)); }},
      {"sim.startup_delay_ms", [&](auto& k, auto& v) { sc.sim.startup_delay_ms = num(k, v); }},
      {"cost.alpha", [&](auto& k, auto& v) { sc.cost.alpha = num(k, v); }},
      {"cost.beta", [&](auto& k, auto& v) { sc.cost.beta = num(k, v); }},
      {"cost.gamma_w", [&](auto& k, auto& v) { sc.cost.gamma_w = num(k, v); }},
      {"cost.gamma_r", [&](auto& k, auto& v) { sc.cost.gamma_r = num(k, v); }},
      {"exec.kappa_graph_ms", [&](auto& k, auto& v) { sc.overheads.kappa_graph_ms = num(k, v); }},
      {"exec.kappa_std_ms", [&](auto& k, auto& v) { sc.overheads.kappa_std_ms = num(k, v); }},
      {"exec.eta", [&](auto& k, auto& v) { sc.overheads.eta = num(k, v); }},
      {"roofline.p_peak", [&](auto& k, auto& v) { sc.roofline.p_peak = num(k, v); }},
      {"roofline.b_mem", [&](auto& k, auto& v) { sc.roofline.b_mem = num(k, v); }},
      {"roofline.bytes_per_token", [&](auto& k, auto& v) { sc.roofline.bytes_per_token = num(k, v); }},
      {"roofline.ops_per_token", [&](auto& k, auto& v) { sc.roofline.ops_per_token = num(k, v); }},
      {"sched.w_min_ms", [&](auto& k, auto& v) { sc.sched.w_min_ms = num(k, v); }},
      {"sched.w_max_ms", [&](auto& k, auto& v) { sc.sched.w_max_ms = num(k, v); }},
      {"sched.sigma_ms", [&](auto& k, auto& v) { sc.sched.sigma_ms = num(k, v); }},
      {"sched.delta_ms", [&](auto& k, auto& v) { sc.sched.delta_ms = num(k, v); }},
      {"sched.t_max_ms", [&](auto& k, auto& v) { sc.sched.t_max_ms = num(k, v); }},
      {"sched.epsilon_per_ms", [&](auto& k, auto& v) { sc.sched.epsilon_per_ms = num(k, v); }},
      {"sched.m_s_tokens", [&](auto& k, auto& v) { sc.sched.m_s_tokens = integer(k, v); }},
      {"sched.c_l_tokens", [&](auto& k, auto& v) { sc.sched.c_l_tokens = integer(k, v); }},
      {"sched.mode",
       [&](auto&, auto& v) {
         if (v == "sla") sc.sched.mode = SchedMode::kSla;
         else if (v == "deadline_free") sc.sched.mode = SchedMode::kDeadlineFree;
         else throw ConfigError("sched.mode: expected sla or deadline_free");
       }},
      {"sched.l_m_first", [&](auto& k, auto& v) { sc.sched.l_m_first = integer(k, v); }},
      {"sched.l_m_re", [&](auto& k, auto& v) { sc.sched.l_m_re = integer(k, v); }},
      {"sched.s_hat_init_ms", [&](auto& k, auto& v) { sc.sched.s_hat_init_ms = num(k, v); }},
      {"sched.ewma_decay", [&](auto& k, auto& v) { sc.sched.ewma_decay = num(k, v); }},
      {"grid.lengths", [&](auto& k, auto& v) { sc.grid.lengths = int_list<Tokens>(k, v); }},
      {"grid.depths", [&](auto& k, auto& v) { sc.grid.depths = int_list<int>(k, v); }},
      {"grid.mem_per_graph_mb", [&](auto& k, auto& v) { sc.grid.mem_per_graph_bytes = num(k, v) * 1024 * 1024; }},
      {"grid.mem_budget_mb", [&](auto& k, auto& v) { sc.grid.mem_budget_bytes = num(k, v) * 1024 * 1024; }},
      {"ctrl.dt_ms", [&](auto& k, auto& v) { sc.ctrl.dt_ms = num(k, v); }},
      {"ctrl.t_cool_ms", [&](auto& k, auto& v) { sc.ctrl.t_cool_ms = num(k, v); }},
      {"ctrl.tau_hyst", [&](auto& k, auto& v) { sc.ctrl.tau_hyst = num(k, v); }},
      {"ctrl.n_min", [&](auto& k, auto& v) { sc.ctrl.n_min = static_cast<int>(integer(k, v)); }},
      {"ctrl.w_q", [&](auto& k, auto& v) { sc.ctrl.w_q = num(k, v); }},
      {"ctrl.w_e", [&](auto& k, auto& v) { sc.ctrl.w_e = num(k, v); }},
      {"ctrl.w_u", [&](auto& k, auto& v) { sc.ctrl.w_u = num(k, v); }},
      {"ctrl.percentile", [&](auto& k, auto& v) { sc.ctrl.aggregator_percentile = static_cast<int>(integer(k, v)); }},
      {"trace.path", [&](auto&, auto& v) { sc.trace_path = v; }},
  };
  for (const auto& [key, v] : cfg) {
    if (key == "grid.model_preset") continue;
    if (auto it = keys.find(key); it != keys.end()) {
      it->second(key, v);
      continue;
    }
    const size_t dot = key.find('.');
    const std::string sect = dot == std::string::npos ? key : key.substr(0, dot);
    const std::string sub = dot == std::string::npos ? "" : key.substr(dot + 1);
    if (sect == "workload" && set_synth(sc.workload, sub, key, v)) continue;
    if (sect == "workload2") {
      if (!sc.workload2) sc.workload2.emplace();
      if (sub == "shift_ms") {
        sc.workload2_shift_ms = num(key, v);
        continue;
      }
      if (set_synth(*sc.workload2, sub, key, v)) continue;
    }
    throw ConfigError("unknown config key: " + key);
  }
  return sc;
}

std::vector<Request> build_workload(const Scenario& sc) {
  if (sc.trace_path) return load_trace(*sc.trace_path);
  std::vector<Request> reqs = synth_stream(sc.workload, sc.workload.duration_ms.value_or(sc.sim.duration_ms));
  if (sc.workload2) {
    const double shift = sc.workload2_shift_ms;
    const double dur2 = sc.workload2->duration_ms.value_or(std::max(0.0, sc.sim.duration_ms - shift));
    reqs = merge_streams(std::move(reqs), shift_stream(synth_stream(*sc.workload2, dur2), shift));
  }
  return reqs;
}

void apply_sweep_param(ConfigMap& cfg, const std::string& param, double value) {
  auto fmt = [](double x) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", x);
    return std::string(buf);
  };
  if (param == "short_concurrency" || param == "long_concurrency") {
    const std::string key = param == "short_concurrency" ? "workload.lambda_per_ms" : "workload2.lambda_per_ms";
    double base = SynthConfig{}.lambda_per_ms;
    if (auto it = cfg.find(key); it != cfg.end()) base = num(key, it->second);
    cfg[key] = fmt(base * value);
    return;
  }
  cfg[param] = fmt(value);
}

RunResult run_scenario(const Scenario& sc) {
  const std::vector<Request> reqs = build_workload(sc);
  return run(sc.sim, reqs, sc.cost, sc.overheads, sc.sched, sc.grid, sc.ctrl);
}

}  // namespace laps
