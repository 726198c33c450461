// The prefill tier: lanes (one per prefill instance / GPU) pulling batches
// from the length-aware queues, driven either by a virtual clock or by the
// wall clock.
//
// Behavioural contract (not structure): for the same config the virtual-clock
// run emits the reference simulator's events.log byte for byte
// (/root/reference/proj/src/sim.cpp:63-669; tests/test_host_engine.py pins 15
// scenarios). That fixes the order in which events are handled — (time,
// insertion order), arrivals before the requests they enable, lanes visited
// in id order — and the floating-point expressions of the clock, nothing else.
//
// Design:
//   Agenda     timed events (arrivals, window wake-ups, startup readiness,
//              controller ticks and — virtual clock only — completions).
//   Lane       one instance: its pool, its AWD state, the job it runs, the
//              long prompt it is chunking, the controller's counters.
//   Router     what a policy means: which queue a request joins, which lanes
//              serve it, what an idle lane does next.
//   Journal    the LogRecord stream (events.log) with sequence numbers.
//   Tier       owns the above and the ForwardBackend every forward goes to.
// Clocks:
//   kVirtual   completion = launch time + the backend's service time (closed
//              form, or a measured GPU time in LIVE mode), scheduled on the
//              agenda — the reference's discrete-event semantics.
//   kWall      time is steady_clock since start; arrivals are released when
//              their time comes, completions are whatever the backend
//              reports finished (CUDA events), so TTFT includes every host
//              and device cost. Several lanes' forwards run concurrently.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <unordered_map>

#include "laps_host.hpp"

namespace laps {

Policy parse_policy(const std::string& s) {
  static const std::pair<const char*, Policy> kNames[] = {
      {"laps", Policy::kLaps}, {"fcfs_unified", Policy::kFcfsUnified}, {"bucket_no_disagg", Policy::kBucketNoDisagg}};
  for (const auto& [name, p] : kNames)
    if (s == name) return p;
  throw ConfigError("sim.policy: '" + s + "' is not one of laps, fcfs_unified, bucket_no_disagg");
}

Disagg parse_disagg(const std::string& s) {
  if (s == "temporal") return Disagg::kTemporal;
  if (s == "spatial") return Disagg::kSpatial;
  throw ConfigError("sim.disagg: '" + s + "' is neither temporal nor spatial");
}

const char* to_string(Policy p) {
  switch (p) {
    case Policy::kLaps: return "laps";
    case Policy::kFcfsUnified: return "fcfs_unified";
    case Policy::kBucketNoDisagg: return "bucket_no_disagg";
  }
  return "?";
}

const char* to_string(Disagg d) { return d == Disagg::kSpatial ? "spatial" : "temporal"; }

void validate(const SimConfig& c) {
  const bool laps = c.policy == Policy::kLaps;
  struct Rule {
    bool broken;
    const char* why;
  };
  const Rule rules[] = {
      {c.n_instances < 1, "sim.instances must be >= 1"},
      {laps && c.disagg == Disagg::kSpatial && c.n_instances < 2,
       "spatial disaggregation needs a short and a long pool (sim.instances >= 2)"},
      {laps && c.disagg == Disagg::kTemporal && c.n_instances != 1,
       "temporal disaggregation shares one instance between both classes (sim.instances = 1)"},
      {c.controller_on && !(laps && c.disagg == Disagg::kSpatial), "sim.controller only applies to spatial pools"},
      {!(c.duration_ms >= 0), "sim.duration_ms must be >= 0"},
      {!(c.slo_ms > 0), "sim.slo_ms must be > 0"},
      {c.unified_token_budget < 1, "sim.unified_token_budget must be >= 1"},
      {c.unified_max_batch < 1, "sim.unified_max_batch must be >= 1"},
      {c.startup_delay_ms < 0, "sim.startup_delay_ms must be >= 0"},
  };
  for (const Rule& r : rules)
    if (r.broken) throw ConfigError(r.why);
}

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

// ------------------------------------------------------------------ agenda
enum class Tick : std::uint8_t { kArrival, kWake, kDone, kReady, kControl };

struct Due {
  double t;
  std::int64_t order;  // insertion order breaks time ties
  Tick what;
  int lane;
  size_t req;
};

class Agenda {
 public:
  void at(double t, Tick what, int lane, size_t req = 0) {
    heap_.push_back(Due{t, order_++, what, lane, req});
    std::push_heap(heap_.begin(), heap_.end(), later);
  }
  bool empty() const { return heap_.empty(); }
  const Due& next() const { return heap_.front(); }
  Due take() {
    std::pop_heap(heap_.begin(), heap_.end(), later);
    Due d = heap_.back();
    heap_.pop_back();
    return d;
  }

 private:
  static bool later(const Due& a, const Due& b) { return a.t > b.t || (a.t == b.t && a.order > b.order); }
  std::vector<Due> heap_;
  std::int64_t order_ = 0;
};

// -------------------------------------------------------------------- lanes
// What a lane is running. `slots` is the AWD depth the service time is
// spread over when the per-slot estimate S_hat learns from it.
struct Job {
  ForwardKind kind = ForwardKind::kAwdBatch;
  std::vector<RequestId> ids;
  const char* cls = "short";
  double service_ms = 0;
  int chunk = 0, chunks = 0;
  bool completes = true;  // final chunk (or not chunked): members get their TTFT
  int slots = 0;
  std::uint64_t handle = 0;
};

// A long prompt being prefilled chunk by chunk, back to back on one lane.
struct ChunkChain {
  Request req;
  std::vector<ChunkDesc> parts;
  size_t next = 0;
  bool active = false;
  bool exhausted() const { return next >= parts.size(); }
};

struct Lane {
  int id = 0;
  PoolKind pool = PoolKind::kShort;
  bool busy = false;
  double busy_from = 0;  // start of the current forward (or startup)
  AwdState awd;
  Job job;
  ChunkChain chain;
  // Controller window counters (reset every tick).
  double busy_ms = 0;
  double late_ms = 0;
  std::int64_t finished = 0;
};

// ------------------------------------------------------------------- router
// The four serving disciplines of the reference, as one value.
enum class Discipline { kUnifiedFcfs, kBucketed, kLapsTemporal, kLapsSpatial };

Discipline discipline_of(const SimConfig& s) {
  switch (s.policy) {
    case Policy::kFcfsUnified: return Discipline::kUnifiedFcfs;
    case Policy::kBucketNoDisagg: return Discipline::kBucketed;
    case Policy::kLaps: break;
  }
  return s.disagg == Disagg::kTemporal ? Discipline::kLapsTemporal : Discipline::kLapsSpatial;
}

struct Queues {
  std::deque<Request> shorts, longs, unified;
  bool any() const { return !shorts.empty() || !longs.empty() || !unified.empty(); }
};

// ------------------------------------------------------------------ journal
class Journal {
 public:
  LogRecord& open(EventKind k, double t) {
    LogRecord& r = recs_.emplace_back();
    r.kind = k;
    r.t = t;
    r.seq = static_cast<std::int64_t>(recs_.size()) - 1;
    return r;
  }
  std::vector<LogRecord> take() { return std::move(recs_); }

 private:
  std::vector<LogRecord> recs_;
};

// --------------------------------------------------------------------- tier
class Tier {
 public:
  Tier(const SimConfig& sim, const std::vector<Request>& reqs, const CostParams& cost, const ExecOverheads& ov,
       const SchedConfig& sched, const GraphGrid& grid, const ControllerConfig& ctrl, ForwardBackend& backend,
       TierClock clock)
      : sim_(sim), reqs_(reqs), cost_(cost), ov_(ov), sched_(sched), grid_(grid), ctrl_(ctrl), fwd_(backend),
        clock_(clock), rule_(discipline_of(sim)) {}

  std::vector<LogRecord> run() {
    check_config();
    build_lanes();
    for (size_t i = 1; i < reqs_.size(); ++i)
      if (reqs_[i].arrival_ms < reqs_[i - 1].arrival_ms)
        throw ConfigError("the request stream must be ordered by arrival time");
    if (!reqs_.empty()) agenda_.at(reqs_[0].arrival_ms, Tick::kArrival, -1, 0);
    if (sim_.controller_on) agenda_.at(ctrl_.dt_ms, Tick::kControl, -1);
    if (clock_ == TierClock::kVirtual) run_virtual();
    else run_wall();
    if (work_left()) throw std::logic_error("engine stopped with requests still queued or in flight");
    fwd_.finish_run();
    return journal_.take();
  }

 private:
  // ---- configuration
  void check_config() const {
    validate(sim_);
    validate(cost_);
    validate(ov_);
    validate(sched_);
    validate(grid_);
    if (!sim_.controller_on) return;
    validate(ctrl_, sim_.n_instances);
    if (ctrl_.n_min < 1) throw ConfigError("ctrl.n_min must be >= 1: the controller may not empty a pool");
  }

  void build_lanes() {
    const int n = sim_.n_instances;
    int shorts = n;
    if (rule_ == Discipline::kLapsSpatial) {
      shorts = sim_.initial_short_instances >= 0 ? sim_.initial_short_instances : (n + 1) / 2;
      const int least = sim_.controller_on ? std::max(1, ctrl_.n_min) : 1;
      if (std::min(shorts, n - shorts) < least)
        throw ConfigError("sim.initial_short_instances leaves the short or long pool below its minimum size");
    }
    lanes_.resize(static_cast<size_t>(n));
    pools_.assignment.clear();
    for (int i = 0; i < n; ++i) {
      Lane& ln = lanes_[static_cast<size_t>(i)];
      ln.id = i;
      ln.pool = i < shorts ? PoolKind::kShort : PoolKind::kLong;
      ln.awd = make_awd_state(sched_, grid_);
      pools_.assignment.push_back(ln.pool);
      if (sim_.startup_delay_ms > 0) {  // graph capture before the lane can serve
        ln.busy = true;
        ln.busy_from = 0;
        agenda_.at(sim_.startup_delay_ms, Tick::kReady, i);
      }
    }
  }

  // ---- clocks
  void handle(const Due& d) {
    switch (d.what) {
      case Tick::kArrival: admit(d.req); break;
      case Tick::kWake: serve_if_idle(lane(d.lane)); break;
      case Tick::kDone: complete(lane(d.lane), lane(d.lane).job.service_ms); break;
      case Tick::kReady: {
        Lane& ln = lane(d.lane);
        charge_busy(ln);
        ln.busy = false;
        serve(ln);
        break;
      }
      case Tick::kControl: control(); break;
    }
  }

  void run_virtual() {
    while (!agenda_.empty()) {
      const Due d = agenda_.take();
      now_ = d.t;
      handle(d);
    }
  }

  double wall_now() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
  }

  // Wall clock: finished forwards first (lane order), then every agenda entry
  // whose time has come; otherwise sleep until the next entry, polling the
  // in-flight forwards every ~20 us.
  void run_wall() {
    t0_ = std::chrono::steady_clock::now();
    for (;;) {
      bool progressed = false;
      for (Lane& ln : lanes_) {
        if (!ln.busy || !in_flight(ln)) continue;
        double ms = 0;
        if (fwd_.poll(ln.job.handle, &ms)) {
          now_ = wall_now();
          ln.job.handle = 0;
          complete(ln, ms);
          progressed = true;
        }
      }
      now_ = wall_now();
      while (!agenda_.empty() && agenda_.next().t <= now_) {
        const Due d = agenda_.take();
        handle(d);
        progressed = true;
      }
      if (progressed) continue;
      const bool flying = std::any_of(lanes_.begin(), lanes_.end(), [&](const Lane& l) { return in_flight(l); });
      if (agenda_.empty() && !flying) break;
      const double until = agenda_.empty() ? kInf : agenda_.next().t - now_;
      const double nap_ms = flying ? std::min(until, 0.02) : until;
      if (nap_ms > 0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(nap_ms));
    }
  }
  bool in_flight(const Lane& ln) const { return ln.busy && ln.job.handle != 0; }

  // ---- arrivals
  bool long_class(const Request& r) const {
    return classify(r, sched_.l_m_first, sched_.l_m_re) == LengthClass::kLong;
  }
  std::deque<Request>& queue_for(bool is_long) {
    if (rule_ == Discipline::kUnifiedFcfs || rule_ == Discipline::kBucketed) return queues_.unified;
    return is_long ? queues_.longs : queues_.shorts;
  }
  // Lanes that may run a request of this class.
  bool eligible(const Lane& ln, bool is_long) const {
    if (rule_ != Discipline::kLapsSpatial) return true;
    return ln.pool == (is_long ? PoolKind::kLong : PoolKind::kShort);
  }
  // Arrivals that feed the AWD arrival-rate estimate of open rounds.
  bool feeds_awd(bool is_long) const {
    return rule_ == Discipline::kBucketed ||
           ((rule_ == Discipline::kLapsTemporal || rule_ == Discipline::kLapsSpatial) && !is_long);
  }

  void admit(size_t idx) {
    const Request& r = reqs_[idx];
    const bool lng = long_class(r);
    {
      // Wall clock: the request arrived at its scheduled time, whatever the
      // engine's lag in noticing it (TTFT is measured from there).
      LogRecord& rec = journal_.open(EventKind::kArrival, clock_ == TierClock::kWall ? r.arrival_ms : now_);
      rec.req = r.id;
      rec.cls = lng ? "long" : "short";
      rec.length = r.new_tokens;
      rec.history = r.history_tokens;
      rec.deadline_ms = r.deadline_ms;
    }
    arrival_of_[r.id] = r.arrival_ms;
    released_ = idx + 1;
    if (released_ < reqs_.size()) agenda_.at(reqs_[released_].arrival_ms, Tick::kArrival, -1, released_);
    queue_for(lng).push_back(r);
    if (feeds_awd(lng))
      for (Lane& ln : lanes_)
        if (eligible(ln, lng) && ln.awd.round_open) ++ln.awd.arrivals_in_round;
    for (Lane& ln : lanes_)
      if (eligible(ln, lng)) serve_if_idle(ln);
  }

  // ---- what an idle lane does next (the length-aware router)
  void serve_if_idle(Lane& ln) {
    if (!ln.busy) serve(ln);
  }

  void serve(Lane& ln) {
    if (ln.busy) return;
    switch (rule_) {
      case Discipline::kUnifiedFcfs:
        pack(ln);
        return;
      case Discipline::kBucketed:
        form_batch(ln, queues_.unified);
        return;
      case Discipline::kLapsSpatial:
        if (ln.pool == PoolKind::kShort) form_batch(ln, queues_.shorts);
        else start_chain(ln);
        return;
      case Discipline::kLapsTemporal: {
        // One lane, two classes: the older head-of-line goes first (ties to
        // short); when the short batcher decides to keep waiting, the lane
        // fills the gap with long work.
        auto& s = queues_.shorts;
        auto& l = queues_.longs;
        if (s.empty() && l.empty()) return;
        const bool short_first = !s.empty() && (l.empty() || s.front().arrival_ms <= l.front().arrival_ms);
        if (!short_first || !form_batch(ln, s)) {
          if (!l.empty()) start_chain(ln);
        }
        return;
      }
    }
  }

  // AWD (SLA) or token-budget admission over a short queue; dispatches a
  // batch or arms the lane's wake-up.
  bool form_batch(Lane& ln, std::deque<Request>& q) {
    const AwdDecision dec = sched_.mode == SchedMode::kSla ? awd_step(ln.awd, q, now_, grid_, sched_)
                                                           : token_max_admit(ln.awd, q, now_, grid_, sched_);
    if (!dec.plan) {
      if (std::isfinite(dec.next_check_ms)) agenda_.at(std::max(dec.next_check_ms, now_), Tick::kWake, ln.id);
      return false;
    }
    dispatch_plan(ln, *dec.plan, q);
    return true;
  }

  static std::vector<Request> take_members(std::deque<Request>& q, const std::vector<RequestId>& ids) {
    std::unordered_map<RequestId, size_t> rank;
    for (size_t k = 0; k < ids.size(); ++k) rank.emplace(ids[k], k);
    std::vector<Request> out(ids.size());
    std::deque<Request> rest;
    for (Request& r : q) {
      auto it = rank.find(r.id);
      if (it != rank.end()) out[it->second] = std::move(r);
      else rest.push_back(std::move(r));
    }
    q.swap(rest);
    return out;
  }

  const char* class_label(const std::vector<Request>& members) const {
    int longs = 0;
    for (const Request& r : members) longs += long_class(r) ? 1 : 0;
    if (longs == 0) return "short";
    return longs == static_cast<int>(members.size()) ? "long" : "mixed";
  }

  static ForwardCall call_for(int lane, double now, ForwardKind kind, BatchShape shape,
                              const std::vector<Request>& members) {
    ForwardCall c;
    c.inst = lane;
    c.now_ms = now;
    c.kind = kind;
    c.shape = shape;
    for (const Request& r : members)
      c.rows.push_back(ForwardRow{r.id, r.session_id, r.new_tokens, r.history_tokens, true});
    return c;
  }

  void dispatch_plan(Lane& ln, const BatchPlan& plan, std::deque<Request>& q) {
    const std::vector<Request> members = take_members(q, plan.members);
    ForwardCall call = call_for(ln.id, now_, ForwardKind::kAwdBatch, plan.shape, members);
    // The closed form bills every row at l_pad, dummy rows up to the depth too.
    std::vector<MemberShape> billed;
    billed.reserve(static_cast<size_t>(std::max<int>(plan.shape.depth, static_cast<int>(members.size()))));
    for (const Request& r : members) billed.emplace_back(r.new_tokens, r.history_tokens);
    billed.resize(std::max(billed.size(), static_cast<size_t>(plan.shape.depth)), MemberShape{0, 0});
    call.model_service_ms = batch_service_time(plan.shape, billed, cost_, ov_);

    Job job;
    job.kind = ForwardKind::kAwdBatch;
    job.ids = plan.members;
    job.cls = class_label(members);
    job.slots = static_cast<int>(members.size());
    launch(ln, call, std::move(job), [&](LogRecord& rec) {
      rec.reason = to_string(plan.reason);
      rec.l_pad = plan.shape.l_pad;
      rec.depth = plan.shape.depth;
      rec.graph = plan.shape.kind == ShapeKind::kGraph;
      rec.real_tokens = plan.real_tokens;
      rec.padded_tokens = plan.shape.l_pad * plan.shape.depth;
    });
  }

  // Long prompts: pop the head of the long queue and prefill it as C_l-token
  // chunks back to back on this lane.
  bool start_chain(Lane& ln) {
    if (queues_.longs.empty()) return false;
    ChunkChain& ch = ln.chain;
    ch.req = queues_.longs.front();
    queues_.longs.pop_front();
    ch.parts = long_chunk_dispatch(ch.req, sched_);
    ch.next = 0;
    ch.active = true;
    next_chunk(ln);
    return true;
  }

  void next_chunk(Lane& ln) {
    ChunkChain& ch = ln.chain;
    const ChunkDesc part = ch.parts[ch.next++];
    const BatchShape shape{part.tokens, 1, ShapeKind::kStandard};
    ForwardCall call;
    call.inst = ln.id;
    call.now_ms = now_;
    call.kind = ForwardKind::kLongChunk;
    call.shape = shape;
    call.rows.push_back(ForwardRow{ch.req.id, ch.req.session_id, part.tokens, part.history, ch.exhausted()});
    const MemberShape row{part.tokens, part.history};
    call.model_service_ms = batch_service_time(shape, std::span<const MemberShape>(&row, 1), cost_, ov_);

    Job job;
    job.kind = ForwardKind::kLongChunk;
    job.ids = {ch.req.id};
    job.cls = "long";
    job.chunk = part.index;
    job.chunks = static_cast<int>(ch.parts.size());
    job.completes = ch.exhausted();
    job.slots = 1;
    launch(ln, call, std::move(job), [&](LogRecord& rec) {
      rec.reason = "long_chunk";
      rec.l_pad = part.tokens;
      rec.depth = 1;
      rec.graph = false;
      rec.real_tokens = rec.padded_tokens = part.tokens;
      rec.chunk = part.index;
      rec.chunks_total = static_cast<int>(ch.parts.size());
    });
  }

  // FCFS baseline: the longest FIFO prefix under the token budget and batch
  // cap (the head always goes), packed without padding.
  void pack(Lane& ln) {
    auto& q = queues_.unified;
    if (q.empty()) return;
    const size_t cap = static_cast<size_t>(sim_.unified_max_batch);
    size_t n = 1;
    Tokens sum = q.front().new_tokens;
    for (; n < q.size() && n < cap && sum + q[n].new_tokens <= sim_.unified_token_budget; ++n) sum += q[n].new_tokens;
    std::vector<Request> members(std::make_move_iterator(q.begin()), std::make_move_iterator(q.begin() + static_cast<long>(n)));
    q.erase(q.begin(), q.begin() + static_cast<long>(n));
    Tokens longest = 0;
    std::vector<MemberShape> rows;
    std::vector<RequestId> ids;
    for (const Request& r : members) {
      longest = std::max(longest, r.new_tokens);
      rows.emplace_back(r.new_tokens, r.history_tokens);
      ids.push_back(r.id);
    }
    const BatchShape shape{longest, static_cast<int>(n), ShapeKind::kStandard};
    ForwardCall call = call_for(ln.id, now_, ForwardKind::kPacked, shape, members);
    call.model_service_ms = packed_service_time(rows, cost_, ov_);

    Job job;
    job.kind = ForwardKind::kPacked;
    job.ids = std::move(ids);
    job.cls = class_label(members);
    job.slots = static_cast<int>(n);
    launch(ln, call, std::move(job), [&](LogRecord& rec) {
      rec.reason = "fcfs_pack";
      rec.l_pad = longest;
      rec.depth = static_cast<int>(n);
      rec.graph = false;
      rec.real_tokens = rec.padded_tokens = sum;  // packed: nothing padded
    });
  }

  // Every forward goes through here: hand it to the backend, log the
  // dispatch, occupy the lane until the forward completes.
  template <typename Fields>
  void launch(Lane& ln, const ForwardCall& call, Job job, Fields&& fields) {
    job.handle = fwd_.launch(call);
    if (clock_ == TierClock::kVirtual) job.service_ms = fwd_.clock_ms(job.handle, call);
    LogRecord& rec = journal_.open(EventKind::kDispatch, now_);
    rec.inst = ln.id;
    rec.reqs = job.ids;
    rec.cls = job.cls;
    fields(rec);
    ln.busy = true;
    ln.busy_from = now_;
    ln.job = std::move(job);
    if (clock_ == TierClock::kVirtual) {
      ln.job.handle = 0;
      agenda_.at(now_ + ln.job.service_ms, Tick::kDone, ln.id);
    } else if (ln.job.handle == 0) {
      throw std::logic_error("wall-clock runs need a backend that returns forward handles");
    }
  }

  // ---- completion
  void complete(Lane& ln, double service_ms) {
    charge_busy(ln);
    Job job = std::move(ln.job);
    job.service_ms = service_ms;
    {
      LogRecord& rec = journal_.open(EventKind::kBatchComplete, now_);
      rec.inst = ln.id;
      rec.reqs = job.ids;
      rec.cls = job.cls;
      rec.service_ms = service_ms;
      rec.chunk = job.chunk;
      rec.chunks_total = job.chunks;
      rec.final_chunk = job.completes;
    }
    if (job.kind == ForwardKind::kAwdBatch) observe_service(ln.awd, service_ms, job.slots, sched_);
    if (job.completes) {
      for (RequestId id : job.ids) {
        ln.late_ms += std::max(0.0, now_ - arrival_of_.at(id) - sim_.slo_ms);
        ++ln.finished;
      }
    }
    ln.busy = false;
    if (ln.chain.active) {
      if (!ln.chain.exhausted()) return next_chunk(ln);  // back to back, no routing decision
      ln.chain.active = false;
      ln.chain.parts.clear();
    }
    serve(ln);
  }

  // ---- Alg. 2 pool controller
  void charge_busy(Lane& ln) { ln.busy_ms += now_ - std::max(ln.busy_from, period_from_); }

  void control() {
    const double dt = ctrl_.dt_ms;
    const int n_s = pools_.n_short(), n_l = pools_.n_long();
    std::vector<double> score(lanes_.size());
    std::vector<double> by_pool[2];
    for (Lane& ln : lanes_) {
      if (ln.busy) charge_busy(ln);
      const bool in_short = ln.pool == PoolKind::kShort;
      InstanceStats st;
      st.u = std::clamp(ln.busy_ms / dt, 0.0, 1.0);
      st.e = ln.finished > 0 ? ln.late_ms / static_cast<double>(ln.finished) : 0.0;
      st.q = static_cast<double>(in_short ? queues_.shorts.size() : queues_.longs.size()) /
             static_cast<double>(in_short ? n_s : n_l);
      score[static_cast<size_t>(ln.id)] = pressure(st, ctrl_);
      by_pool[in_short ? 0 : 1].push_back(score[static_cast<size_t>(ln.id)]);
      ln.busy_ms = ln.late_ms = 0;
      ln.finished = 0;
    }
    const double p_s = aggregate(by_pool[0], ctrl_.aggregator_percentile);
    const double p_l = aggregate(by_pool[1], ctrl_.aggregator_percentile);
    const std::optional<MigrationDir> move = decide(p_s, p_l, pools_, ctrl_, now_);
    Lane* donor = nullptr;
    if (move) {
      // The least pressured lane of the pool that gives one up changes sides;
      // its open AWD round is abandoned, an in-flight forward drains first.
      const PoolKind from = *move == MigrationDir::kLongToShort ? PoolKind::kLong : PoolKind::kShort;
      for (Lane& ln : lanes_)
        if (ln.pool == from && (!donor || score[static_cast<size_t>(ln.id)] < score[static_cast<size_t>(donor->id)]))
          donor = &ln;
      donor->pool = from == PoolKind::kLong ? PoolKind::kShort : PoolKind::kLong;
      pools_.assignment[static_cast<size_t>(donor->id)] = donor->pool;
      donor->awd.round_open = false;
      donor->awd.arrivals_in_round = 0;
      donor->awd.next_check = kInf;
    }
    {
      LogRecord& tick = journal_.open(EventKind::kControllerTick, now_);
      tick.n_short = pools_.n_short();
      tick.n_long = pools_.n_long();
      tick.p_short = p_s;
      tick.p_long = p_l;
      tick.migrated = donor != nullptr;
    }
    if (donor) {
      LogRecord& m = journal_.open(EventKind::kMigration, now_);
      m.inst = donor->id;
      m.direction = to_string(*move);
      m.n_short = pools_.n_short();
      m.n_long = pools_.n_long();
      serve_if_idle(*donor);
    }
    period_from_ = now_;
    if (work_left()) agenda_.at(now_ + dt, Tick::kControl, -1);
  }

  bool work_left() const {
    return released_ < reqs_.size() || queues_.any() ||
           std::any_of(lanes_.begin(), lanes_.end(), [](const Lane& l) { return l.busy; });
  }
  Lane& lane(int i) { return lanes_[static_cast<size_t>(i)]; }

  const SimConfig sim_;
  const std::vector<Request>& reqs_;
  const CostParams cost_;
  const ExecOverheads ov_;
  const SchedConfig sched_;
  const GraphGrid grid_;
  const ControllerConfig ctrl_;
  ForwardBackend& fwd_;
  const TierClock clock_;
  const Discipline rule_;

  std::vector<Lane> lanes_;
  Queues queues_;
  Agenda agenda_;
  Journal journal_;
  PoolState pools_;
  std::unordered_map<RequestId, double> arrival_of_;
  size_t released_ = 0;  // requests admitted so far
  double now_ = 0;
  double period_from_ = 0;  // start of the controller's current window
  std::chrono::steady_clock::time_point t0_;
};

}  // namespace

RunResult run_tier(const SimConfig& sim, const std::vector<Request>& requests, const CostParams& cost,
                   const ExecOverheads& overheads, const SchedConfig& sched, const GraphGrid& grid,
                   const ControllerConfig& ctrl, ForwardBackend& backend, TierClock clock) {
  Tier tier(sim, requests, cost, overheads, sched, grid, ctrl, backend, clock);
  RunResult out;
  out.log = tier.run();
  out.report = metrics_from_log(out.log, sim.slo_ms);
  return out;
}

RunResult run_with_backend(const SimConfig& sim, const std::vector<Request>& requests, const CostParams& cost,
                           const ExecOverheads& overheads, const SchedConfig& sched, const GraphGrid& grid,
                           const ControllerConfig& ctrl, ForwardBackend& backend) {
  return run_tier(sim, requests, cost, overheads, sched, grid, ctrl, backend, TierClock::kVirtual);
}

RunResult run(const SimConfig& sim, const std::vector<Request>& requests, const CostParams& cost,
              const ExecOverheads& overheads, const SchedConfig& sched, const GraphGrid& grid,
              const ControllerConfig& ctrl) {
  CostModelBackend closed_form;
  return run_tier(sim, requests, cost, overheads, sched, grid, ctrl, closed_form, TierClock::kVirtual);
}

}  // namespace laps
