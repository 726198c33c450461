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
// Nearest-rank percentile: the ceil(q n / 100)-th smallest sample (the 1e-9
// keeps 0.9 * 10 from rounding up to rank 10).
double percentile(std::span<const double> samples, double q) {
  if (samples.empty()) throw EmptySamples();
  if (!(q > 0 && q <= 100)) throw std::invalid_argument("percentile: q must lie in (0, 100]");
  std::vector<double> v(samples.begin(), samples.end());
  const double n = static_cast<double>(v.size());
  size_t rank = static_cast<size_t>(std::ceil(q * n / 100.0 - 1e-9));
  rank = std::min(std::max<size_t>(rank, 1), v.size());
  std::nth_element(v.begin(), v.begin() + static_cast<long>(rank - 1), v.end());
  return v[rank - 1];
}

double slo_violation_rate(std::span<const double> t, double slo_ms) {
  if (t.empty()) throw EmptySamples();
  const auto late = std::count_if(t.begin(), t.end(), [&](double x) { return x > slo_ms; });
  return static_cast<double>(late) / static_cast<double>(t.size());
}

namespace {

// Everything one class (overall / short / long) contributes to metrics.json.
struct ClassBook {
  std::vector<double> ttft, wait;  // per request, in arrival order
  std::int64_t batches = 0, graph_batches = 0, members = 0;
  Tokens real = 0, padded = 0;

  void batch(const LogRecord& r) {
    batches += 1;
    graph_batches += r.graph ? 1 : 0;
    members += static_cast<std::int64_t>(r.reqs.size());
    real += r.real_tokens;
    padded += r.padded_tokens;
  }

  static double mean(const std::vector<double>& v) {
    double acc = 0;
    for (double x : v) acc += x;
    return acc / static_cast<double>(v.size());
  }

  ClassMetrics finish(double slo_ms, double active_ms) const {
    ClassMetrics m;
    m.completed = static_cast<std::int64_t>(ttft.size());
    m.batches = batches;
    if (!ttft.empty()) {
      m.ttft_mean_ms = mean(ttft);
      m.ttft_p50_ms = percentile(ttft, 50);
      m.ttft_p90_ms = percentile(ttft, 90);
      m.ttft_p99_ms = percentile(ttft, 99);
      m.slo_violation = slo_violation_rate(ttft, slo_ms);
      if (active_ms > 0) m.rps = 1000.0 * static_cast<double>(m.completed) / active_ms;
    }
    if (!wait.empty()) m.mean_wait_ms = mean(wait);
    if (batches > 0) {
      const double nb = static_cast<double>(batches);
      m.mean_depth = static_cast<double>(members) / nb;
      m.graph_hit_rate = static_cast<double>(graph_batches) / nb;
    }
    if (real > 0) m.padding_overhead = static_cast<double>(padded) / static_cast<double>(real) - 1.0;
    return m;
  }
};

// One request's milestones on the log's clock (-1 = never happened).
struct Milestones {
  double arrived = 0, dispatched = -1, finished = -1;
  bool is_long = false;
};

}  // namespace

// Metrics are recomputed from the event log alone (the log is the contract):
// arrivals open a request, its first dispatch ends its wait, the completion
// of its final chunk ends its TTFT; RPS counts completions over the span
// from the first arrival to the last completion.
MetricsReport metrics_from_log(std::span<const LogRecord> log, double slo_ms) {
  std::vector<Milestones> reqs;                  // arrival order
  std::unordered_map<RequestId, size_t> where;  // request id -> reqs index
  ClassBook all, shorts, longs;
  MetricsReport rep;
  rep.slo_ms = slo_ms;
  bool seen_arrival = false, seen_completion = false;
  double t_first = 0, t_last = 0;
  auto milestones = [&](RequestId id) -> Milestones* {
    const auto it = where.find(id);
    return it == where.end() ? nullptr : &reqs[it->second];
  };
  for (const LogRecord& r : log) {
    if (r.kind == EventKind::kArrival) {
      where[r.req] = reqs.size();
      reqs.push_back(Milestones{r.t, -1, -1, r.cls == "long"});
      rep.arrivals += 1;
      t_first = seen_arrival ? std::min(t_first, r.t) : r.t;
      seen_arrival = true;
    } else if (r.kind == EventKind::kDispatch) {
      for (RequestId id : r.reqs)
        if (Milestones* m = milestones(id); m && m->dispatched < 0) m->dispatched = r.t;
      all.batch(r);
      if (r.cls == "short") shorts.batch(r);
      else if (r.cls == "long") longs.batch(r);
    } else if (r.kind == EventKind::kBatchComplete && r.final_chunk) {
      for (RequestId id : r.reqs) {
        Milestones* m = milestones(id);
        if (!m) continue;
        m->finished = r.t;
        t_last = seen_completion ? std::max(t_last, r.t) : r.t;
        seen_completion = true;
      }
    } else if (r.kind == EventKind::kMigration) {
      rep.migrations += 1;
    }
  }
  if (seen_arrival && seen_completion && t_last > t_first) rep.active_ms = t_last - t_first;
  for (const Milestones& m : reqs) {
    ClassBook& cls = m.is_long ? longs : shorts;
    if (m.finished >= 0) {
      all.ttft.push_back(m.finished - m.arrived);
      cls.ttft.push_back(m.finished - m.arrived);
    }
    if (m.dispatched >= 0) {
      all.wait.push_back(m.dispatched - m.arrived);
      cls.wait.push_back(m.dispatched - m.arrived);
    }
  }
  rep.overall = all.finish(slo_ms, rep.active_ms);
  rep.short_cls = shorts.finish(slo_ms, rep.active_ms);
  rep.long_cls = longs.finish(slo_ms, rep.active_ms);
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
