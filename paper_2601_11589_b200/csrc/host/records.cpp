// The engine's observable outputs: the JSONL event log (frozen field order and
// %.6f times — the byte-parity artifact, event_log.cpp:55-97 of the reference)
// and metrics recomputed from it (metrics.cpp:15-236: nearest-rank
// percentiles, RPS over first arrival -> last completion, arrival-order sums).
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <fstream>
#include <unordered_map>

#include "laps_host.hpp"

namespace laps {

namespace {

void appendf(std::string& out, const char* fmt, ...) {
  char buf[320];
  va_list ap;
  va_start(ap, fmt);
  const int n = vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  out.append(buf, static_cast<size_t>(std::max(0, std::min<int>(n, sizeof(buf) - 1))));
}

void append_ids(std::string& out, const std::vector<RequestId>& ids) {
  out += '[';
  for (size_t i = 0; i < ids.size(); ++i) {
    if (i) out += ',';
    appendf(out, "%" PRId64, ids[i]);
  }
  out += ']';
}

}  // namespace

const char* to_string(EventKind k) {
  switch (k) {
    case EventKind::kArrival: return "arrival";
    case EventKind::kDispatch: return "dispatch";
    case EventKind::kBatchComplete: return "batch_complete";
    case EventKind::kControllerTick: return "controller_tick";
    case EventKind::kMigration: return "migration";
  }
  return "?";
}

std::string serialize(const LogRecord& r) {
  std::string s;
  s.reserve(192);
  appendf(s, "{\"t\":%.6f,\"seq\":%" PRId64 ",\"kind\":\"%s\"", r.t, r.seq, to_string(r.kind));
  if (r.kind == EventKind::kArrival) {
    appendf(s, ",\"req\":%" PRId64 ",\"cls\":\"%s\",\"L\":%" PRId64 ",\"H\":%" PRId64, r.req, r.cls.c_str(),
            r.length, r.history);
    if (r.deadline_ms) appendf(s, ",\"ddl\":%.6f", *r.deadline_ms);
  } else if (r.kind == EventKind::kDispatch) {
    appendf(s, ",\"inst\":%d,\"reqs\":", r.inst);
    append_ids(s, r.reqs);
    appendf(s, ",\"cls\":\"%s\",\"reason\":\"%s\",\"l_pad\":%" PRId64 ",\"depth\":%d,\"graph\":%d", r.cls.c_str(),
            r.reason.c_str(), r.l_pad, r.depth, r.graph ? 1 : 0);
    appendf(s, ",\"real\":%" PRId64 ",\"padded\":%" PRId64 ",\"chunk\":%d,\"chunks\":%d", r.real_tokens,
            r.padded_tokens, r.chunk, r.chunks_total);
  } else if (r.kind == EventKind::kBatchComplete) {
    appendf(s, ",\"inst\":%d,\"reqs\":", r.inst);
    append_ids(s, r.reqs);
    appendf(s, ",\"cls\":\"%s\",\"service\":%.6f,\"chunk\":%d,\"chunks\":%d,\"final\":%d", r.cls.c_str(),
            r.service_ms, r.chunk, r.chunks_total, r.final_chunk ? 1 : 0);
  } else if (r.kind == EventKind::kControllerTick) {
    appendf(s, ",\"n_s\":%d,\"n_l\":%d,\"p_s\":%.6f,\"p_l\":%.6f,\"migrated\":%d", r.n_short, r.n_long,
            r.p_short, r.p_long, r.migrated ? 1 : 0);
  } else {
    appendf(s, ",\"inst\":%d,\"dir\":\"%s\",\"n_s\":%d,\"n_l\":%d", r.inst, r.direction.c_str(), r.n_short,
            r.n_long);
  }
  s += '}';
  return s;
}

void write_event_log(const std::string& path, std::span<const LogRecord> log) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path);
  for (const auto& r : log) out << serialize(r) << '\n';
}

// ------------------------------------------------------------------ metrics
double percentile(std::span<const double> samples, double q) {
  if (samples.empty()) throw EmptySamples();
  if (!(q > 0) || q > 100) throw std::invalid_argument("percentile rank must be in (0, 100]");
  std::vector<double> v(samples.begin(), samples.end());
  std::sort(v.begin(), v.end());
  // rank = ceil(q*n/100), nudged so 0.9*10 does not round up to 10.
  const double n = static_cast<double>(v.size());
  const size_t rank = std::clamp<size_t>(static_cast<size_t>(std::ceil(q * n / 100.0 - 1e-9)), 1, v.size());
  return v[rank - 1];
}

double slo_violation_rate(std::span<const double> t, double slo_ms) {
  if (t.empty()) throw EmptySamples();
  std::int64_t over = 0;
  for (double x : t) over += x > slo_ms ? 1 : 0;
  return static_cast<double>(over) / static_cast<double>(t.size());
}

namespace {

struct Tally {
  std::int64_t batches = 0, graph = 0, depth = 0;
  Tokens real = 0, padded = 0;
  void add(const LogRecord& r) {
    ++batches;
    graph += r.graph ? 1 : 0;
    depth += static_cast<std::int64_t>(r.reqs.size());
    real += r.real_tokens;
    padded += r.padded_tokens;
  }
};

ClassMetrics summarise(const std::vector<double>& ttft, const std::vector<double>& wait, const Tally& b,
                       double slo_ms, double active_ms) {
  ClassMetrics m;
  m.completed = static_cast<std::int64_t>(ttft.size());
  if (!ttft.empty()) {
    double sum = 0;
    for (double t : ttft) sum += t;
    m.ttft_mean_ms = sum / static_cast<double>(ttft.size());
    m.ttft_p50_ms = percentile(ttft, 50);
    m.ttft_p90_ms = percentile(ttft, 90);
    m.ttft_p99_ms = percentile(ttft, 99);
    m.slo_violation = slo_violation_rate(ttft, slo_ms);
    if (active_ms > 0) m.rps = 1000.0 * static_cast<double>(m.completed) / active_ms;
  }
  if (!wait.empty()) {
    double sum = 0;
    for (double w : wait) sum += w;
    m.mean_wait_ms = sum / static_cast<double>(wait.size());
  }
  m.batches = b.batches;
  if (b.batches > 0) {
    m.mean_depth = static_cast<double>(b.depth) / static_cast<double>(b.batches);
    m.graph_hit_rate = static_cast<double>(b.graph) / static_cast<double>(b.batches);
  }
  if (b.real > 0) m.padding_overhead = static_cast<double>(b.padded) / static_cast<double>(b.real) - 1.0;
  return m;
}

}  // namespace

MetricsReport metrics_from_log(std::span<const LogRecord> log, double slo_ms) {
  struct Info {
    double arrival = 0, first_dispatch = -1, completion = -1;
    bool is_long = false;
  };
  MetricsReport rep;
  rep.slo_ms = slo_ms;
  std::unordered_map<RequestId, Info> info;
  std::vector<RequestId> order;
  Tally all, shorts, longs;
  double first_arrival = std::numeric_limits<double>::infinity();
  double last_completion = -std::numeric_limits<double>::infinity();
  for (const auto& r : log) {
    switch (r.kind) {
      case EventKind::kArrival:
        info[r.req] = Info{r.t, -1, -1, r.cls == "long"};
        order.push_back(r.req);
        rep.arrivals += 1;
        first_arrival = std::min(first_arrival, r.t);
        break;
      case EventKind::kDispatch:
        for (RequestId id : r.reqs) {
          auto it = info.find(id);
          if (it != info.end() && it->second.first_dispatch < 0) it->second.first_dispatch = r.t;
        }
        all.add(r);
        if (r.cls == "short") shorts.add(r);
        if (r.cls == "long") longs.add(r);
        break;
      case EventKind::kBatchComplete:
        if (!r.final_chunk) break;
        for (RequestId id : r.reqs) {
          auto it = info.find(id);
          if (it != info.end()) {
            it->second.completion = r.t;
            last_completion = std::max(last_completion, r.t);
          }
        }
        break;
      case EventKind::kMigration:
        rep.migrations += 1;
        break;
      case EventKind::kControllerTick:
        break;
    }
  }
  if (std::isfinite(first_arrival) && last_completion > first_arrival) rep.active_ms = last_completion - first_arrival;
  std::vector<double> t_all, t_s, t_l, w_all, w_s, w_l;
  for (RequestId id : order) {  // arrival order keeps double sums reproducible
    const Info& ri = info.at(id);
    if (ri.completion >= 0) {
      const double t = ri.completion - ri.arrival;
      t_all.push_back(t);
      (ri.is_long ? t_l : t_s).push_back(t);
    }
    if (ri.first_dispatch >= 0) {
      const double w = ri.first_dispatch - ri.arrival;
      w_all.push_back(w);
      (ri.is_long ? w_l : w_s).push_back(w);
    }
  }
  rep.overall = summarise(t_all, w_all, all, slo_ms, rep.active_ms);
  rep.short_cls = summarise(t_s, w_s, shorts, slo_ms, rep.active_ms);
  rep.long_cls = summarise(t_l, w_l, longs, slo_ms, rep.active_ms);
  return rep;
}

std::string to_json(const MetricsReport& m) {
  std::string o = "{\n";
  appendf(o, "  \"slo_ms\": %.6f,\n", m.slo_ms);
  appendf(o, "  \"active_ms\": %.6f,\n", m.active_ms);
  appendf(o, "  \"arrivals\": %" PRId64 ",\n", m.arrivals);
  appendf(o, "  \"migrations\": %" PRId64 ",\n", m.migrations);
  const std::pair<const char*, const ClassMetrics*> classes[] = {
      {"overall", &m.overall}, {"short", &m.short_cls}, {"long", &m.long_cls}};
  for (int k = 0; k < 3; ++k) {
    const ClassMetrics& c = *classes[k].second;
    appendf(o, "  \"%s\": {\n", classes[k].first);
    appendf(o, "    \"completed\": %" PRId64 ",\n", c.completed);
    appendf(o, "    \"ttft_mean_ms\": %.6f,\n", c.ttft_mean_ms);
    appendf(o, "    \"ttft_p50_ms\": %.6f,\n", c.ttft_p50_ms);
    appendf(o, "    \"ttft_p90_ms\": %.6f,\n", c.ttft_p90_ms);
    appendf(o, "    \"ttft_p99_ms\": %.6f,\n", c.ttft_p99_ms);
    appendf(o, "    \"rps\": %.6f,\n", c.rps);
    appendf(o, "    \"slo_violation\": %.6f,\n", c.slo_violation);
    appendf(o, "    \"mean_wait_ms\": %.6f,\n", c.mean_wait_ms);
    appendf(o, "    \"batches\": %" PRId64 ",\n", c.batches);
    appendf(o, "    \"mean_depth\": %.6f,\n", c.mean_depth);
    appendf(o, "    \"graph_hit_rate\": %.6f,\n", c.graph_hit_rate);
    appendf(o, "    \"padding_overhead\": %.6f\n", c.padding_overhead);
    o += k < 2 ? "  },\n" : "  }\n";
  }
  o += "}\n";
  return o;
}

void write_metrics(const std::string& path, const MetricsReport& m) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path);
  out << to_json(m);
}

}  // namespace laps
