#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>

#include "abi_common.h"
#include "executor.h"
#include "attn_plan.h"
#include "launch.cuh"

#include <nvtx3/nvToolsExt.h>

namespace lp {

namespace {

constexpr int kPage = kAttnPage;  // 64 tokens per KV page (== attention key tile)
constexpr int kAttnSplitExtra = 2 * 148;  // extra attention work items for key-range splits

// Tensor ids for the counter-based weight generator (oracle/forward_oracle.py
// uses the same numbering).
constexpr uint64_t kTidEmbed = 1, kTidLmHead = 2;
constexpr uint64_t kTidLayerBase = 1000, kTidLayerStride = 16;
enum : uint64_t { kQkv = 0, kQkvBias = 1, kO = 2, kGate = 3, kUp = 4, kDown = 5 };

template <typename T>
T* dmalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) {
    throw OutOfMemory("cudaMalloc " + std::to_string(n * sizeof(T)) + " bytes: " +
                      cudaGetErrorString(e));
  }
  owned.push_back(p);
  return static_cast<T*>(p);
}

int pow2_bn(int t) {
  int b = 16;
  while (b < t && b < 256) b <<= 1;
  return b;
}

// Largest split-K factor a launch capacity allows: >= 4 k-blocks per split,
// S * t_cap <= 8192 rows of fp32 partials (workspace bound), S <= 8.
int split_cap(int K, int t_cap) { return std::max(1, std::min({8, (K / 64) / 4, std::max(1, 8192 / t_cap)})); }

}  // namespace

// Split-K factor minimising wave quantisation for the LIVE token count:
// time ~ ceil(units*S/workers)/S per unit of work, with a small charge per
// extra split for the fp32 partial round trip.
int choose_splits(int M, int bn, int pair, int n_live, int s_cap, int sms) {
  const int workers = sms / pair;
  const int units = (M / (128 * pair)) * std::max(1, (n_live + bn - 1) / bn);
  int best_s = 1;
  double best = 1e30;
  for (int s = 1; s <= s_cap; ++s) {
    const double waves = static_cast<double>((units * s + workers - 1) / workers);
    const double cost = waves / s * (1.0 + 0.03 * (s - 1));
    if (cost < best - 1e-9) {
      best = cost;
      best_s = s;
    }
  }
  return best_s;
}

// Measured per-tile cost of a narrow token tile on B200 (7B projections at
// T = 4096, forced tile counts): a tile of width tw costs ~ (tw + 55..105)
// columns' worth of time (TMA issue, MMA issue, accumulator hand-off).
constexpr double kTileOverheadCols = 80.0;

// Per-batch (token tiles, split-K) plan. Weight-streaming batches (< 256 live
// tokens) keep ceil(n/bn) tiles and the wave-quantisation split choice. For
// tensor-bound batches the plan minimises an estimate in microseconds:
//   waves * (tile width + kTileOverheadCols) * (K-blocks per split + 2) * kUsPerColKb
//   + (S - 1) * M * n_live * 8 B / partial bandwidth
// — every extra split writes one more fp32 partial of the output in the GEMM
// and the reduction kernel (qkv_post / resid_rmsnorm) reads it back. Tile
// widths are multiples of 16 (the MMA N is a runtime operand). The constants
// are fitted to the tile sweeps of profiles/r02_tile_sweep.txt (32B QKV at 512
// tokens: 1 split 32.8 us; the former +3 %-per-split charge chose 5 splits and
// made the reduction read 73 MB of partials instead of 15).
constexpr double kUsPerColKb = 1.19e-3;  // one tile column x one 64-deep K block, per CTA (pair)
static double partial_bytes_per_us() {
  static const double v = [] {
    const char* e = std::getenv("LP_PARTIAL_GBS");  // experiments: effective partial bandwidth, GB/s
    return (e ? std::atof(e) : 4000.0) * 1e3;
  }();
  return v;
}

// Stream-K (split-K-capable GEMMs, tensor-bound batches): groups of nt CTAs
// (pairs) take equal shares `per` of the m_tiles x nk (weight tile, K-block)
// steps, one token tile per member, so a one-wave GEMM (32B QKV / O at 512 tokens: 56 /
// 40 tiles on 74 pairs) keeps every SM busy. Estimate: (per + 2 per segment)
// steps at the tile width, plus the partial traffic: one extra fp32 tile per
// share boundary, written by the GEMM and read back by the reduction kernel.
static int stream_k_mode() {
  static const int v = [] {
    const char* e = std::getenv("LP_STREAMK");  // experiments: 0 = split-K plans only, 2 = stream-K wherever it fits
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// Stream-K share of one worker group (one CTA (pair) per token tile, the
// groups splitting the m_tiles x nk (weight tile, K-block) steps), and the
// largest segment count of any tile; 0 groups: not runnable.
long sk_share(int m_tiles, int n_tiles, int nk, int workers) {
  const int groups = workers / n_tiles;
  return groups < 1 ? 0 : (long(m_tiles) * nk + groups - 1) / groups;
}
int sk_max_segments(int m_tiles, int n_tiles, int nk, int workers) {
  const long per = sk_share(m_tiles, n_tiles, nk, workers);
  return per < 1 ? 1 << 20 : int((nk - 1) / per) + 2;
}

// CTA (pair) count of a launch: the grid gemm_launch sizes for the plan's
// capacity (s_cap x m_tiles x nt_cap units, at most one per SM (pair)).
int gemm_workers(int M, const GemmPlan& p, int sms) {
  const long units = long(std::max(1, p.s_cap)) * (M / (128 * p.pair)) * p.nt_cap;
  return int(std::min<long>(sms / p.pair, units));
}

TilePlan choose_tiles(int M, int K, const GemmPlan& p, int n_live, int sms) {
  TilePlan t;
  const int base = std::max(1, (n_live + p.bn - 1) / p.bn);
  t.n_tiles = base;
  if (n_live < 256) {
    t.splits = choose_splits(M, p.bn, p.pair, n_live, p.s_cap, sms);
    return t;
  }
  const int workers = sms / p.pair, m_tiles = M / (128 * p.pair), nk = K / 64;
  const int nt_hi = std::min(p.nt_cap, (n_live + 15) / 16);
  const int grid_workers = gemm_workers(M, p, sms);
  double best = 1e30;
  for (int nt = base; nt <= nt_hi; ++nt) {
    const int tw = ((n_live + nt - 1) / nt + 15) / 16 * 16;
    if (nt > base && (nt - 1) * tw >= n_live) continue;  // same widths as a smaller count
    for (int s = 1; s <= p.s_cap; ++s) {
      const long units = long(m_tiles) * nt * s;
      const double waves = static_cast<double>((units + workers - 1) / workers);
      const double cost = waves * (tw + kTileOverheadCols) * (double(nk) / s + 2.0) * kUsPerColKb +
                          double(s - 1) * M * n_live * 8.0 / partial_bytes_per_us();
      if (cost < best * (1 - 1e-9)) {
        best = cost;
        t.n_tiles = nt;
        t.splits = s;
        t.stream_k = false;
      }
    }
    // Stream-K candidate: every tile's segments must fit the workspace slices.
    // Measured to pay only between one and three 256-token tiles (deep-K
    // down projections; profiles/r02_stream_k.txt), so it is offered there.
    const int skm = stream_k_mode();
    if (p.s_cap >= 2 && ((n_live > 256 && n_live <= 768 && skm == 1) || skm == 2) &&
        sk_max_segments(m_tiles, nt, nk, grid_workers) <= p.s_cap) {
      const long per = sk_share(m_tiles, nt, nk, grid_workers);
      const double segs = double((per + nk - 1) / nk + 1);
      const double extra = double(grid_workers - 1) * 128.0 * p.pair * tw * 8.0;  // partial bytes (bound)
      const double cost = skm == 2 ? -1.0
                                   : (double(per) + 2.0 * segs) * (tw + kTileOverheadCols) * kUsPerColKb +
                                         extra / partial_bytes_per_us();
      if (skm == 2 ? !t.stream_k : cost < best * (1 - 1e-9)) {
        best = cost;
        t.n_tiles = nt;
        t.splits = 1;
        t.stream_k = true;
      }
    }
  }
  return t;
}

namespace {

// bn: smallest power-of-two tile >= tokens (<= 256). CTA pairs
// (cta_group::2) once the token tile is >= 128 wide: the activation tile is
// then re-read per 256 weight rows instead of per 128. Split-K (fp32-partial
// outputs only) is chosen per batch from the live token count at submit time
// (device metadata); `splits` here is the choice at full capacity.
GemmPlan plan_gemm(int M, int K, int t_cap, bool allow_split, int sms) {
  GemmPlan p;
  p.bn = pow2_bn(std::min(t_cap, 256));
  p.pair = (p.bn >= 128 && M % 256 == 0) ? 2 : 1;
  const int base_nt = (t_cap + p.bn - 1) / p.bn;
  p.nt_cap = t_cap >= 256 ? std::min(4 * base_nt, (t_cap + 15) / 16) : base_nt;
  if (!allow_split) return p;
  p.s_cap = split_cap(K, t_cap);
  p.splits = choose_splits(M, p.bn, p.pair, t_cap, p.s_cap, sms);
  return p;
}

}  // namespace

Instance::Instance(const lp_model_desc& m, const lp_instance_desc& d) : m_(m), d_(d) {
  if (m.head_dim != 64 && m.head_dim != 128) throw ConfigError("head_dim must be 64 or 128");
  if (m.n_q_heads % m.n_kv_heads != 0) throw ConfigError("n_q_heads % n_kv_heads != 0");
  if (m.hidden % 128 || ((m.n_q_heads + 2 * m.n_kv_heads) * m.head_dim) % 128 ||
      (2 * m.intermediate) % 128 || m.vocab % 128 || m.intermediate % 64)
    throw ConfigError("model dims must be multiples of 128 (hidden, qkv, 2*intermediate, vocab)");
  if (d.page_size != 0 && d.page_size != kPage) throw ConfigError("page_size must be 64");
  d_.page_size = kPage;
  if (d_.max_tokens <= 0) d_.max_tokens = 16384;
  if (d_.max_members <= 0) d_.max_members = 64;
  if (d_.max_members > 65535) throw ConfigError("max_members must be <= 65535 (attention work items pack the member index in 16 bits)");
  if (const char* e = std::getenv("LP_FUSE_EPI")) {  // "1" both, "qkv", "resid"
    const std::string v(e);
    fuse_qkv_ = v == "1" || v == "qkv";
    fuse_resid_ = v == "1" || v == "resid";
  }
  if (const char* e = std::getenv("LP_GRAPH_ATTN_TC_MIN")) graph_tc_min_ = std::atoi(e);
  if (const char* e = std::getenv("LP_GRAPH_TC_PAIRS")) graph_tc_pairs_ = std::atoll(e);
  if (const char* e = std::getenv("LP_ATTN_TC"); e && e[0] == '0') attn_tc_ = false;
  if (const char* e = std::getenv("LP_ATTN_PERSIST"); e && e[0] == '0') attn_persist_ = false;
  lp_check(cudaSetDevice(d.device), "cudaSetDevice");
  lp_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  lp_check(cudaEventCreate(&ev_start_), "event");
  lp_check(cudaEventCreate(&ev_end_), "event");
  lp_check(cudaEventCreateWithFlags(&ev_mig_, cudaEventDisableTiming), "event");
  lp_check(cudaEventCreateWithFlags(&ev_mig_done_, cudaEventDisableTiming), "event");
  for (Staging& sg : staging_) lp_check(cudaEventCreateWithFlags(&sg.h2d, cudaEventDisableTiming), "event");
  for (Ticket& tk : tickets_) {
    lp_check(cudaEventCreate(&tk.start), "event");
    lp_check(cudaEventCreate(&tk.end), "event");
    lp_check(cudaEventCreateWithFlags(&tk.done, cudaEventDisableTiming), "event");
  }
  alloc_weights();
  alloc_arena();
}

Instance::~Instance() {
  cudaSetDevice(d_.device);
  cudaStreamSynchronize(stream_);
  for (auto& [k, g] : graphs_) cudaGraphExecDestroy(g);
  for (auto& [k, g] : graphs_nc_) cudaGraphExecDestroy(g);
  for (auto& [k, g] : graphs_tc_) cudaGraphExecDestroy(g);
  for (auto& [k, g] : chunk_graphs_) cudaGraphExecDestroy(g);
  for (void* p : allocs_) cudaFree(p);
  if (mig_host_) cudaFreeHost(mig_host_);
  for (Staging& sg : staging_) {
    if (sg.host) cudaFreeHost(sg.host);
    cudaEventDestroy(sg.h2d);
  }
  for (Ticket& tk : tickets_) {
    if (tk.keys) cudaFreeHost(tk.keys);
    cudaEventDestroy(tk.start);
    cudaEventDestroy(tk.end);
    cudaEventDestroy(tk.done);
  }
  cudaEventDestroy(ev_start_);
  cudaEventDestroy(ev_end_);
  cudaEventDestroy(ev_mig_);
  cudaEventDestroy(ev_mig_done_);
  for (cudaEvent_t e : timers_)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(stream_);
}

void Instance::alloc_weights() {
  const int h = m_.hidden, I = m_.intermediate, D = m_.head_dim;
  const int qkv_out = (m_.n_q_heads + 2 * m_.n_kv_heads) * D;
  const int o_in = m_.n_q_heads * D;
  const float scale = m_.init_std * std::sqrt(3.0f) / 8388608.0f;  // U(-a,a), a = std*sqrt(3)
  const uint64_t seed = m_.weight_seed;
  cudaStream_t st = stream_;
  layers_.resize(m_.layers);
  for (int l = 0; l < m_.layers; ++l) {
    LayerW& w = layers_[l];
    const uint64_t base = kTidLayerBase + kTidLayerStride * l;
    w.wqkv = dmalloc<bf16>(size_t(qkv_out) * h, allocs_);
    w.bqkv = dmalloc<bf16>(qkv_out, allocs_);
    w.wo = dmalloc<bf16>(size_t(h) * o_in, allocs_);
    w.wgu = dmalloc<bf16>(size_t(2) * I * h, allocs_);
    w.wd = dmalloc<bf16>(size_t(h) * I, allocs_);
    w.g_attn = dmalloc<bf16>(h, allocs_);
    w.g_mlp = dmalloc<bf16>(h, allocs_);
    init_weights(w.wqkv, size_t(qkv_out) * h, seed, base + kQkv, scale, 0, h, st);
    init_weights(w.bqkv, qkv_out, seed, base + kQkvBias, scale, 0, 1, st);
    init_weights(w.wo, size_t(h) * o_in, seed, base + kO, scale, 0, o_in, st);
    init_weights(w.wgu, size_t(2) * I * h, seed, base + kGate, scale, /*interleave*/ 1, h, st);
    init_weights(w.wd, size_t(h) * I, seed, base + kDown, scale, 0, I, st);
    fill_bf16(w.g_attn, h, 1.0f, st);
    fill_bf16(w.g_mlp, h, 1.0f, st);
    w.tm_qkv = make_tmap_bf16(w.wqkv, qkv_out, h, 128);
    w.tm_o = make_tmap_bf16(w.wo, h, o_in, 128);
    w.tm_gu = make_tmap_bf16(w.wgu, 2 * I, h, 128);
    w.tm_d = make_tmap_bf16(w.wd, h, I, 128);
  }
  embed_ = dmalloc<bf16>(size_t(m_.vocab) * h, allocs_);
  lm_head_ = dmalloc<bf16>(size_t(m_.vocab) * h, allocs_);
  g_final_ = dmalloc<bf16>(h, allocs_);
  // Embedding rows ~ U(-sqrt3, sqrt3) (unit variance) so the residual stream
  // starts O(1); every other tensor uses init_std.
  init_weights(embed_, size_t(m_.vocab) * h, seed, kTidEmbed, std::sqrt(3.0f) / 8388608.0f, 0, h, st);
  init_weights(lm_head_, size_t(m_.vocab) * h, seed, kTidLmHead, scale, 0, h, st);
  fill_bf16(g_final_, h, 1.0f, st);
  tm_lm_ = make_tmap_bf16(lm_head_, m_.vocab, h, 128);

  std::vector<float> inv(D / 2);
  for (int i = 0; i < D / 2; ++i)
    inv[i] = static_cast<float>(1.0 / std::pow(static_cast<double>(m_.rope_theta), (2.0 * i) / D));
  inv_freq_ = dmalloc<float>(D / 2, allocs_);
  lp_check(cudaMemcpyAsync(inv_freq_, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice, st), "inv_freq");
  lp_check(cudaGetLastError(), "weight init");
  lp_check(cudaStreamSynchronize(st), "weight init sync");
}

void Instance::alloc_arena() {
  const int h = m_.hidden, I = m_.intermediate, D = m_.head_dim;
  const int qkv_out = (m_.n_q_heads + 2 * m_.n_kv_heads) * D;
  const int G = m_.n_q_heads / m_.n_kv_heads;
  t_max_ = static_cast<int>(d_.max_tokens);
  r_max_ = d_.max_members;
  c_max_ = (t_max_ * G + kAttnRows - 1) / kAttnRows + r_max_;
  w_max_ = c_max_ + kAttnSplitExtra;
  // Persistent pieces: every (128-row block, kv head) unit plus one split per CTA boundary.
  pw_max_ = ((t_max_ * G + kAttnTcRows - 1) / kAttnTcRows + r_max_) * m_.n_kv_heads + 2 * kAttnMaxCtas;

  x_resid_ = dmalloc<float>(size_t(t_max_) * h, allocs_);
  x_norm_ = dmalloc<bf16>(size_t(t_max_) * h, allocs_);
  q_ = dmalloc<bf16>(size_t(t_max_) * m_.n_q_heads * D, allocs_);
  attn_ = dmalloc<bf16>(size_t(t_max_) * m_.n_q_heads * D, allocs_);
  act_ = dmalloc<bf16>(size_t(t_max_) * I, allocs_);
  x_last_ = dmalloc<bf16>(size_t(std::max(r_max_, 256)) * h, allocs_);
  logits_ = dmalloc<float>(size_t(r_max_) * m_.vocab, allocs_);
  next_keys_ = dmalloc<unsigned long long>(r_max_, allocs_);

  // Split-K workspace: max over every capacity we may launch with.
  ws_elems_ = 0;
  for (int t = 16; t <= t_max_; t += 16) {
    const SplitPlan p = plan_for(t, 1);
    const size_t mx = std::max<size_t>({size_t(p.qkv.s_cap) * qkv_out, size_t(p.o.s_cap) * h,
                                        size_t(p.d.s_cap) * h});
    ws_elems_ = std::max(ws_elems_, mx * size_t(t));
  }
  ws_ = dmalloc<float>(ws_elems_, allocs_);
  // Stream-K segment table (kSkTab*): one int per (128-row tile, 16-token tile) bounds it.
  {
    const size_t n = kSkTabHeader + size_t(std::max(qkv_out, h)) / 128 * size_t((t_max_ + 15) / 16);
    sk_tab_ = dmalloc<int>(n, allocs_);
    lp_check(cudaMemset(sk_tab_, 0, n * sizeof(int)), "memset sk table");
  }

  // KV pool.
  page_elems_ = size_t(2) * m_.n_kv_heads * kPage * D;
  const size_t page_bytes_all = page_elems_ * 2 * m_.layers;
  n_pages_ = d_.kv_pages;
  if (n_pages_ <= 0) {
    size_t fr = 0, tot = 0;
    lp_check(cudaMemGetInfo(&fr, &tot), "meminfo");
    const size_t reserve = size_t(6) << 30;
    n_pages_ = fr > reserve ? static_cast<int64_t>((fr - reserve) / page_bytes_all) : 0;
    n_pages_ = std::min<int64_t>(n_pages_, 1 << 20);
  }
  if (n_pages_ < 1) throw OutOfMemory("no HBM left for the KV pool");
  layer_stride_ = page_elems_ * size_t(n_pages_);
  kv_pool_ = dmalloc<bf16>(layer_stride_ * m_.layers, allocs_);
  for (int32_t p = 0; p < n_pages_; ++p) free_pages_.insert(free_pages_.end(), p);
  // Page-id lists of an incoming session migration (source ids, then ours).
  mig_ids_ = dmalloc<int>(size_t(2) * n_pages_, allocs_);
  lp_check(cudaMallocHost(reinterpret_cast<void**>(&mig_host_), size_t(2) * n_pages_ * sizeof(int)), "pinned ids");
  tm_kv_ = make_kv_tmap(kv_pool_, int64_t(m_.layers) * n_pages_ * 2 * m_.n_kv_heads, D);
  // Key-range split partials: only the first kAttnSplitCap work items may be partial.
  // Eager launches (long chunks, off-grid / packed batches: long key ranges,
  // many rows) use the tcgen05 kernel; graph replays (<= 256 new tokens per
  // member) keep the lighter warp-MMA kernel, whose per-CTA fixed cost is
  // lower for one or two key tiles. The kernel is fixed at capture time.
  attn_rows_ = (D == 128 && attn_tc_) ? kAttnTcRows : kAttnRows;
  attn_ws_o_ = dmalloc<float>(size_t(kAttnSplitCap) * m_.n_kv_heads * attn_rows_ * D, allocs_);
  attn_ws_ml_ = dmalloc<float>(size_t(kAttnSplitCap) * m_.n_kv_heads * attn_rows_ * 2, allocs_);
  const size_t n_tickets = size_t(std::max(c_max_, pw_max_)) * m_.n_kv_heads;
  attn_comb_cnt_ = dmalloc<int>(n_tickets, allocs_);
  lp_check(cudaMemsetAsync(attn_comb_cnt_, 0, n_tickets * sizeof(int), stream_), "tickets");
  max_pages_ = static_cast<int>(std::min<int64_t>(n_pages_, 4096));

  // Metadata block: device + pinned host mirror with identical layout.
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_sc = carve(16 * 4), o_tok = carve(size_t(t_max_) * 4), o_pos = carve(size_t(t_max_) * 4),
               o_slot = carve(size_t(t_max_) * 4), o_qs = carve(r_max_ * 4), o_ql = carve(r_max_ * 4),
               o_h = carve(r_max_ * 4), o_li = carve(r_max_ * 4), o_po = carve(r_max_ * 4),
               o_pt = carve(size_t(r_max_) * max_pages_ * 4), o_w = carve(size_t(std::max(w_max_, pw_max_)) * 16),
               o_cb = carve(size_t(std::max(c_max_, pw_max_)) * 16), o_w2 = carve(size_t(pw_max_) * 16),
               o_co = carve(size_t(kAttnMaxCtas + 1) * 4);
  meta_bytes_ = off;
  meta_dev_ = dmalloc<uint8_t>(meta_bytes_, allocs_);
  auto bind = [&](void* base, Meta& m) {
    uint8_t* b = static_cast<uint8_t*>(base);
    m.scalars = reinterpret_cast<int*>(b + o_sc);
    m.tokens = reinterpret_cast<int*>(b + o_tok);
    m.positions = reinterpret_cast<int*>(b + o_pos);
    m.slots = reinterpret_cast<int*>(b + o_slot);
    m.q_start = reinterpret_cast<int*>(b + o_qs);
    m.q_len = reinterpret_cast<int*>(b + o_ql);
    m.hist = reinterpret_cast<int*>(b + o_h);
    m.last_idx = reinterpret_cast<int*>(b + o_li);
    m.page_table = reinterpret_cast<int*>(b + o_pt);
    m.page_off = reinterpret_cast<int*>(b + o_po);
    m.work = reinterpret_cast<int4*>(b + o_w);
    m.combine = reinterpret_cast<int4*>(b + o_cb);
    m.work2 = reinterpret_cast<int4*>(b + o_w2);
    m.cta_off = reinterpret_cast<int*>(b + o_co);
  };
  bind(meta_dev_, md_);
  for (Staging& sg : staging_) {
    lp_check(cudaMallocHost(&sg.host, meta_bytes_), "pinned meta");
    std::memset(sg.host, 0, meta_bytes_);
    bind(sg.host, sg.m);
  }
  mh_ = staging_[0].m;
  for (Ticket& tk : tickets_)
    lp_check(cudaMallocHost(reinterpret_cast<void**>(&tk.keys), size_t(r_max_) * sizeof(unsigned long long)),
             "pinned first tokens");
  lp_check(cudaMemsetAsync(meta_dev_, 0, meta_bytes_, stream_), "meta zero");
  lp_check(cudaStreamSynchronize(stream_), "arena sync");
}

// Attention grid capacities for a forward launched at (t_cap, r_cap): one
// item per 64-row block of (token, q-head) rows of each member, plus room for
// key-range splits of short batches over long histories.
int Instance::combine_cap_for(int t_cap, int r_cap) const {
  const int G = m_.n_q_heads / m_.n_kv_heads;
  // A row block is split only when the unsplit grid fills at most half of
  // the split target (<= 2 resident CTAs per SM), i.e. blocks * nkv <= SMs:
  // no more than SMs / nkv blocks can need a combine.
  const int split_blocks = (num_sms() + m_.n_kv_heads - 1) / m_.n_kv_heads;
  return std::min({c_max_, (t_cap * G + kAttnRows - 1) / kAttnRows + r_cap, split_blocks});
}
int Instance::block_cap_for(int t_cap, int r_cap) const {
  const int G = m_.n_q_heads / m_.n_kv_heads;
  return std::min(c_max_, (t_cap * G + kAttnRows - 1) / kAttnRows + r_cap);
}
int Instance::work_cap_for(int t_cap, int r_cap) const {
  // Splits only ever target ~2 waves of (items x kv heads) CTAs, so the extra
  // room is 2 * SMs / nkv items (early-exit CTAs beyond the live count still
  // occupy SM slots and would delay the next GEMM's PDL weight prefetch).
  const int extra = std::min(kAttnSplitExtra, (2 * num_sms() + m_.n_kv_heads - 1) / m_.n_kv_heads);
  return std::min(w_max_, block_cap_for(t_cap, r_cap) + extra);
}

GemmPlan plan_gemm_for_tests(int M, int K, int t_cap, bool allow_split, int sms) {
  return plan_gemm(M, K, t_cap, allow_split, sms);
}

SplitPlan Instance::plan_for(int t_cap, int r_cap) const {
  const int sms = num_sms();
  const int h = m_.hidden, D = m_.head_dim;
  const int qkv_out = (m_.n_q_heads + 2 * m_.n_kv_heads) * D;
  SplitPlan p;
  p.qkv = plan_gemm(qkv_out, h, t_cap, true, sms);
  p.o = plan_gemm(h, m_.n_q_heads * D, t_cap, true, sms);
  p.gu = plan_gemm(2 * m_.intermediate, h, t_cap, false, sms);
  p.d = plan_gemm(h, m_.intermediate, t_cap, true, sms);
  p.lm = plan_gemm(m_.vocab, h, std::max(r_cap, 1), false, sms);
  return p;
}

const CUtensorMap& Instance::act_map(const bf16* buf, int rows, int cols, int box_rows) {
  auto key = std::make_tuple(static_cast<const void*>(buf), cols, box_rows);
  auto it = act_maps_.find(key);
  if (it != act_maps_.end()) return it->second;
  return act_maps_.emplace(key, make_tmap_bf16(buf, rows, cols, box_rows)).first->second;
}

void Instance::gemm(const CUtensorMap& tm_w, const GemmPlan& p, GemmArgs g, const bf16* x, int x_rows,
                    cudaStream_t st) {
  // With a device-side split count the grid is sized for the largest one allowed.
  g.splits = g.splits_dev ? p.s_cap : p.splits;
  g.n_tiles_cap = p.nt_cap;
  if (g.splits_dev && g.mode == kEpiF32Partial) g.sk_tab = sk_tab_;  // metadata may select stream-K
  gemm_launch(tm_w, act_map(x, x_rows, g.K, gemm_b_box_rows(p.bn, p.pair)), g, p.bn, st, 0, p.pair);
}

void Instance::enqueue_forward(int t_cap, int r_cap, cudaStream_t st, bool graph, bool combine) {
  const int attn_rows = attn_rows_for(graph, t_cap);
  const int h = m_.hidden, I = m_.intermediate, D = m_.head_dim;
  const int nq = m_.n_q_heads, nkv = m_.n_kv_heads;
  const int qkv_out = (nq + 2 * nkv) * D;
  const SplitPlan p = plan_for(t_cap, r_cap);
  const int* n_tok = md_.scalars + 0;
  const int* n_mem = md_.scalars + 1;
  const RowCtx rc{n_tok, t_cap, h, m_.rms_eps};
  const int G = nq / nkv;
  // Without the merge grid no item is split: the grid needs no split room.
  const int work_cap = combine ? work_cap_for(t_cap, r_cap) : block_cap_for(t_cap, r_cap);
  const int combine_cap = combine_cap_for(t_cap, r_cap);
  (void)G;

  embed_rmsnorm(rc, md_.tokens, embed_, layers_[0].g_attn, x_resid_, x_norm_, st);
  // NVTX: one range per decoder layer of an eager launch / a capture (host
  // side; a graph replay shows up as the caller's "lp_submit" range).
  char layer_tag[32];
  for (int l = 0; l < m_.layers; ++l) {
    std::snprintf(layer_tag, sizeof layer_tag, "layer %d", l);
    nvtxRangePushA(layer_tag);
    const LayerW& w = layers_[l];
    bf16* kv_layer = kv_pool_ + layer_stride_ * l;
    // QKV projection -> fp32 split partials.
    GemmArgs g;
    g.M = qkv_out; g.N = t_cap; g.K = h; g.n_dev = n_tok; g.ntiles_dev = md_.scalars + 8;
    g.mode = kEpiF32Partial; g.ws = ws_; g.ws_stride = t_cap;
    if (fuse_qkv_ && p.qkv.splits == 1 && D == 128) {
      // Bias + RoPE + q / paged-KV writes straight from TMEM (no fp32 round trip).
      g.mode = kEpiQkvRope;
      g.bias = w.bqkv;
      g.qkv = QkvEpi{md_.positions, md_.slots, inv_freq_, q_, kv_layer, nq, nkv, kPage};
      gemm(w.tm_qkv, p.qkv, g, x_norm_, t_max_, st);
    } else {
      g.splits_dev = md_.scalars + 4;  // per-batch split-K (submit)
      gemm(w.tm_qkv, p.qkv, g, x_norm_, t_max_, st);
      QkvCtx qc{n_tok, t_cap, nq, nkv, D, kPage, ws_, p.qkv.splits, md_.scalars + 4, size_t(t_cap), w.bqkv,
                md_.positions, md_.slots, inv_freq_, q_, kv_layer};
      qc.s_cap = p.qkv.s_cap;
      qc.sk_tab = sk_tab_;
      qkv_post(qc, st);
    }
    AttnCtx ac{md_.scalars + 2, md_.work, md_.scalars + 3, md_.combine, md_.q_start, md_.q_len, md_.hist,
               md_.page_table, md_.page_off, q_, static_cast<int>(int64_t(l) * n_pages_ * 2 * nkv), attn_,
               attn_ws_o_, attn_ws_ml_, nq, nkv,
               static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D))), attn_rows,
               attn_comb_cnt_, md_.work2, md_.cta_off};
    if (attn_rows == kAttnTcRows && attn_persist_ && !debug_empty("attn"))
      attention_prefill_tc_persistent(ac, tm_kv_, std::min(num_sms(), kAttnMaxCtas), st);
    else
      attention_prefill(ac, tm_kv_, D, work_cap, combine_cap, st, combine);
    // O projection + residual + RMSNorm.
    g = GemmArgs{};
    g.M = h; g.N = t_cap; g.K = nq * D; g.n_dev = n_tok; g.ntiles_dev = md_.scalars + 9;
    g.mode = kEpiF32Partial; g.ws = ws_; g.ws_stride = t_cap;
    const bool o_fused = fuse_resid_ && p.o.splits == 1;
    if (o_fused) {  // residual add in the epilogue; the norm kernel then reads x_resid only
      g.mode = kEpiResidAdd;
      g.resid = x_resid_;
    } else {
      g.splits_dev = md_.scalars + 5;
    }
    gemm(w.tm_o, p.o, g, attn_, t_max_, st);
    resid_rmsnorm(rc, ws_, 0, o_fused ? nullptr : md_.scalars + 5, sk_tab_, t_cap, x_resid_, w.g_mlp, x_norm_, st);
    // gate/up with fused SiLU*up.
    g = GemmArgs{};
    g.M = 2 * I; g.N = t_cap; g.K = h; g.n_dev = n_tok; g.ntiles_dev = md_.scalars + 10;
    g.mode = kEpiSiluMul; g.out = act_; g.ldo = I;
    gemm(w.tm_gu, p.gu, g, x_norm_, t_max_, st);
    // down + residual + next RMSNorm.
    g = GemmArgs{};
    g.M = h; g.N = t_cap; g.K = I; g.n_dev = n_tok; g.ntiles_dev = md_.scalars + 11;
    g.mode = kEpiF32Partial; g.ws = ws_; g.ws_stride = t_cap;
    const bool d_fused = fuse_resid_ && p.d.splits == 1;
    if (d_fused) {
      g.mode = kEpiResidAdd;
      g.resid = x_resid_;
    } else {
      g.splits_dev = md_.scalars + 6;
    }
    gemm(w.tm_d, p.d, g, act_, t_max_, st);
    const bf16* g_next = (l + 1 < m_.layers) ? layers_[l + 1].g_attn : g_final_;
    resid_rmsnorm(rc, ws_, 0, d_fused ? nullptr : md_.scalars + 6, sk_tab_, t_cap, x_resid_, g_next, x_norm_, st);
    nvtxRangePop();
  }
  // Final norm already applied; LM head on the last real token per member —
  // skipped (0 live rows) when no member wants its first token (an
  // intermediate long-prompt chunk, a history fill).
  const int* n_head = md_.scalars + 12;
  gather_rows(n_head, r_cap, md_.last_idx, x_norm_, x_last_, h, next_keys_, st);
  GemmArgs g;
  g.M = m_.vocab; g.N = r_cap; g.K = h; g.n_dev = n_head;
  g.mode = kEpiF32; g.out = logits_; g.ldo = m_.vocab;
  gemm(tm_lm_, p.lm, g, x_last_, std::max(r_max_, 256), st);
  argmax_rows(n_head, r_cap, logits_, m_.vocab, next_keys_, st);
}

std::vector<int32_t> Instance::alloc_pages(int n) {
  if (static_cast<int64_t>(free_pages_.size()) < n) {
    throw OutOfMemory("KV page pool exhausted (" + std::to_string(free_pages_.size()) +
                      " free, need " + std::to_string(n) + ")");
  }
  std::vector<int32_t> out;
  out.reserve(n);
  for (int i = 0; i < n; ++i) {
    out.push_back(*free_pages_.begin());
    free_pages_.erase(free_pages_.begin());
  }
  return out;
}

void Instance::ensure_capacity(Session& s, int64_t tokens) {
  const int64_t need = (tokens + kPage - 1) / kPage;
  if (need > max_pages_) throw ShapeMismatch("context of " + std::to_string(tokens) + " tokens exceeds page-table capacity");
  if (need > static_cast<int64_t>(s.pages.size())) {
    auto extra = alloc_pages(static_cast<int>(need - s.pages.size()));
    s.pages.insert(s.pages.end(), extra.begin(), extra.end());
  }
}

void Instance::capture_graphs(const std::vector<int64_t>& lens, const std::vector<int32_t>& depths) {
  if (!d_.use_graphs) return;
  lp_check(cudaSetDevice(d_.device), "set device");
  // Warm the launch paths (function attributes, tensor-map cache) eagerly.
  Meta& mh = acquire_staging();
  mh.scalars[0] = mh.scalars[1] = mh.scalars[2] = mh.scalars[3] = 0;
  mh.scalars[12] = 0;
  lp_check(cudaMemcpyAsync(md_.scalars, mh.scalars, 64, cudaMemcpyHostToDevice, stream_), "meta");
  lp_check(cudaEventRecord(staging_[(stage_seq_ - 1) % kStaging].h2d, stream_), "event");
  for (int64_t L : lens) {
    for (int32_t dep : depths) {
      const int64_t t_cap = L * dep;
      if (t_cap > t_max_ || dep > r_max_) continue;
      const int64_t key = graph_key(L, dep);
      if (graphs_.count(key)) continue;
      graphs_[key] = capture_one(static_cast<int>(t_cap), dep, true);
      graphs_nc_[key] = capture_one(static_cast<int>(t_cap), dep, true, false);
      if (m_.head_dim == 128 && attn_tc_) graphs_tc_[key] = capture_one(static_cast<int>(t_cap), dep, false, true);
    }
  }
  for (int t_cap = kChunkGraphStep; t_cap <= std::min(kChunkGraphMax, t_max_); t_cap += kChunkGraphStep)
    if (!chunk_graphs_.count(t_cap)) chunk_graphs_[t_cap] = capture_one(t_cap, 1, false);
  lp_check(cudaStreamSynchronize(stream_), "capture sync");
}

cudaGraphExec_t Instance::capture_one(int t_cap, int r_cap, bool graph_attn, bool combine) {
  enqueue_forward(t_cap, r_cap, stream_, graph_attn, combine);  // warm-up (no live work)
  cudaGraph_t graph;
  lp_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  enqueue_forward(t_cap, r_cap, stream_, graph_attn, combine);
  lp_check(cudaStreamEndCapture(stream_, &graph), "end capture");
  cudaGraphExec_t exec;
  lp_check(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
  cudaGraphDestroy(graph);
  return exec;
}

Meta& Instance::acquire_staging() {
  Staging& sg = staging_[stage_seq_ % kStaging];
  ++stage_seq_;
  if (sg.used) lp_check(cudaEventSynchronize(sg.h2d), "staging reuse");
  sg.used = true;
  mh_ = sg.m;
  return mh_;
}

Instance::Ticket& Instance::ticket(int64_t id) {
  Ticket& tk = tickets_[((id % kTickets) + kTickets) % kTickets];
  if (id < 0 || tk.id != id)
    throw StateError("ticket " + std::to_string(id) + " unknown or expired (results are kept for the last " +
                     std::to_string(kTickets) + " submits)");
  return tk;
}

bool Instance::ticket_done(int64_t id) {
  const cudaError_t e = cudaEventQuery(ticket(id).done);
  if (e == cudaErrorNotReady) return false;
  lp_check(e, "ticket query");
  return true;
}

double Instance::ticket_wait(int64_t id) {
  Ticket& tk = ticket(id);
  lp_check(cudaEventSynchronize(tk.done), "forward");
  float ms = 0;
  lp_check(cudaEventElapsedTime(&ms, tk.start, tk.end), "elapsed");
  return ms;
}

void Instance::ticket_tokens(int64_t id, int32_t* out, int n) {
  Ticket& tk = ticket(id);
  if (n > tk.n) throw ShapeMismatch("asked for more tokens than members");
  lp_check(cudaEventSynchronize(tk.done), "first tokens");
  for (int i = 0; i < n; ++i) out[i] = tk.logits ? argmax_token(tk.keys[i]) : -1;
}

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int64_t Instance::submit(const lp_shape& shape, const lp_member* mem, int n, const int32_t* tokens) {
  const NvtxRange range(shape.kind == LP_KIND_GRAPH ? "lp_submit graph" : shape.kind == LP_KIND_PACKED ? "lp_submit packed" : "lp_submit standard");
  lp_check(cudaSetDevice(d_.device), "set device");
  if (n < 1) throw ShapeMismatch("empty batch");
  if (n > r_max_) throw ShapeMismatch("batch of " + std::to_string(n) + " exceeds max_members");
  if (shape.kind != LP_KIND_PACKED && n > shape.depth)
    throw ShapeMismatch("member count " + std::to_string(n) + " > shape depth " + std::to_string(shape.depth));
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (mem[i].new_tokens < 1) throw ShapeMismatch("member with no new tokens");
    if (shape.kind != LP_KIND_PACKED && mem[i].new_tokens > shape.l_pad)
      throw ShapeMismatch("member length " + std::to_string(mem[i].new_tokens) + " exceeds l_pad " +
                          std::to_string(shape.l_pad));
    total += mem[i].new_tokens;
  }
  if (total > t_max_) throw ShapeMismatch("forward of " + std::to_string(total) + " tokens exceeds arena");

  // Sessions / pages: positions [0, history) must be resident. Positions a
  // member recomputes are overwritten with the same (deterministic) values.
  for (int i = 0; i < n; ++i) {
    Session& s = sessions_[mem[i].session_id];
    if (s.kv_len < mem[i].history) {
      throw std::runtime_error("session " + std::to_string(mem[i].session_id) + ": history " +
                               std::to_string(mem[i].history) + " not resident (have " +
                               std::to_string(s.kv_len) + ")");
    }
    ensure_capacity(s, mem[i].history + mem[i].new_tokens);
  }

  // Results slot of this forward: the ticket kTickets submits ago is dropped
  // (its D2H must have landed before the pinned slot is rewritten).
  const int64_t id = next_ticket_;
  Ticket& tk = tickets_[id % kTickets];
  if (tk.id >= 0) lp_check(cudaEventSynchronize(tk.done), "ticket reuse");
  tk.id = -1;
  // Host metadata, in the next free pinned staging block.
  acquire_staging();
  const int G = m_.n_q_heads / m_.n_kv_heads;
  int t = 0, np = 0;
  for (int i = 0; i < n; ++i) {
    const Session& s = sessions_[mem[i].session_id];
    const int L = static_cast<int>(mem[i].new_tokens), H = static_cast<int>(mem[i].history);
    mh_.q_start[i] = t;
    mh_.q_len[i] = L;
    mh_.hist[i] = H;
    mh_.last_idx[i] = t + L - 1;
    // Ragged page list: only the pages covering [0, H + L) are shipped.
    mh_.page_off[i] = np;
    const int used = (H + L + kPage - 1) / kPage;
    for (int k = 0; k < used; ++k) mh_.page_table[np++] = s.pages[k];
    for (int j = 0; j < L; ++j, ++t) {
      const int pos = H + j;
      mh_.tokens[t] = tokens[t];
      mh_.positions[t] = pos;
      mh_.slots[t] = s.pages[pos / kPage] * kPage + pos % kPage;
    }
  }

  // Which launch runs this batch (fixes the attention grid capacity).
  // Grid-shape graph (warp-MMA attention), chunk graph for a one-member
  // standard launch (tcgen05 attention), else eager sized to the live batch.
  cudaGraphExec_t exec = nullptr;
  bool tc_graph = false;
  int t_cap = std::min(std::max(16, (t + 15) / 16 * 16), t_max_);
  int r_cap = n;
  int attn_rows = attn_rows_;  // matches enqueue_forward
  if (d_.use_graphs && shape.kind == LP_KIND_GRAPH) {
    auto it = graphs_.find(graph_key(shape.l_pad, shape.depth));
    if (it != graphs_.end()) {
      exec = it->second;
      t_cap = static_cast<int>(shape.l_pad * shape.depth);
      r_cap = shape.depth;
      attn_rows = attn_rows_for(true, t_cap);
      int64_t pairs = 0, qtok = 0;
      for (int i = 0; i < n; ++i) {
        pairs += mem[i].new_tokens * (mem[i].history + mem[i].new_tokens);
        qtok += mem[i].new_tokens;
      }
      // tcgen05 pays off for long key ranges (mean keys per query >= 512,
      // i.e. re-prefills over histories) with enough total work; short causal
      // blocks (H = 0) stay on the warp-MMA kernel.
      auto jt = graphs_tc_.find(graph_key(shape.l_pad, shape.depth));
      if (attn_rows != kAttnTcRows && pairs >= graph_tc_pairs_ && pairs >= 512 * qtok && jt != graphs_tc_.end()) {
        exec = jt->second;
        attn_rows = kAttnTcRows;
        tc_graph = true;
      }
    }
  } else if (d_.use_graphs && shape.kind == LP_KIND_STANDARD && n == 1) {
    auto it = chunk_graphs_.find((t + kChunkGraphStep - 1) / kChunkGraphStep * kChunkGraphStep);
    if (it != chunk_graphs_.end()) {
      exec = it->second;
      t_cap = it->first;
      r_cap = 1;
    }
  }
  const int work_cap = work_cap_for(t_cap, r_cap);
  const int combine_cap = combine_cap_for(t_cap, r_cap);

  // Attention work list: one item per 64-row block of (token, q-head) rows;
  // when the blocks cannot fill the GPU, long key ranges are split
  // (>= kMinSplitTiles pages each) and merged by the combine kernel. Split
  // (partial) items come first so their indices address the partial
  // workspace; the rest follow heaviest first.
  struct Blk {
    int r, row0, need;
  };
  std::vector<Blk> blks;
  for (int i = 0; i < n; ++i) {
    const int L = mh_.q_len[i], H = mh_.hist[i];
    for (int r0 = 0; r0 < L * G; r0 += attn_rows) {
      const int p_hi = H + std::min(r0 + attn_rows - 1, L * G - 1) / G;
      blks.push_back({i, r0, (p_hi + 1 + kPage - 1) / kPage});
    }
  }
  std::stable_sort(blks.begin(), blks.end(), [](const Blk& a, const Blk& b) { return a.need > b.need; });
  constexpr int kMinSplitTiles = 2;
  if (attn_rows == kAttnTcRows && attn_persist_) {
    // Persistent tcgen05 attention: balanced piece lists (attn_plan.h).
    const int ncta = std::min(num_sms(), kAttnMaxCtas), nkv = m_.n_kv_heads;
    std::vector<AttnBlock> ab;
    ab.reserve(blks.size());
    for (const Blk& b : blks) ab.push_back(AttnBlock{b.r, b.row0, b.need});
    const AttnSchedule sched = plan_attention(ab, nkv, ncta, size_t(kAttnSplitCap) * nkv);
    std::vector<int4> w1, w2;
    std::vector<int> cta_of;
    for (const AttnPiece& pc : sched.pieces) {
      w1.push_back(make_int4(pc.r, pc.row0, pc.t_begin, pc.t_end));
      w2.push_back(make_int4(pc.g, pc.ci, pc.slot, 0));
      cta_of.push_back(pc.cta);
    }
    int nw = 0;
    const int nc = static_cast<int>(sched.merges.size());
    for (int k = 0; k < nc; ++k) {
      const AttnMerge& m = sched.merges[static_cast<size_t>(k)];
      mh_.combine[k] = make_int4(m.r, m.row0 | m.g << 20, m.first_slot, m.n_pieces);
    }
    if (static_cast<int>(w1.size()) > pw_max_) throw ShapeMismatch("attention schedule exceeds its piece capacity");
    // Counting sort of the pieces by CTA (stable: a CTA keeps creation order).
    std::vector<int> count(kAttnMaxCtas + 1, 0);
    for (int c : cta_of) ++count[static_cast<size_t>(c) + 1];
    for (int c = 0; c < kAttnMaxCtas; ++c) count[static_cast<size_t>(c) + 1] += count[static_cast<size_t>(c)];
    for (int c = 0; c <= kAttnMaxCtas; ++c) mh_.cta_off[c] = count[static_cast<size_t>(c)];
    for (size_t i = 0; i < w1.size(); ++i) {
      const int at = count[static_cast<size_t>(cta_of[i])]++;
      mh_.work[at] = w1[i];
      mh_.work2[at] = w2[i];
    }
    nw = static_cast<int>(w1.size());
    mh_.scalars[2] = nw;
    mh_.scalars[3] = nc;
  } else {
  const int base = static_cast<int>(blks.size());
  // One wave for the tcgen05 kernel (one CTA per SM), two for the warp-MMA one.
  const int ctas = base * m_.n_kv_heads, target = (attn_rows == kAttnTcRows ? 1 : 2) * num_sms();
  // Round DOWN: a split that pushes the grid past one wave of resident CTAs
  // only adds a partial round trip and a combine pass.
  // <= 32 splits for the graph path's merge grid; <= 4 for the tcgen05 kernel,
  // whose last split CTA merges the block itself.
  int f = std::min(attn_rows == kAttnTcRows ? 4 : 32, std::max(1, target / std::max(ctas, 1)));
  if (attn_rows == kAttnTcRows) {
    static const int forced = [] {  // experiments: force the tcgen05 key-split factor
      const char* e = std::getenv("LP_ATTN_TC_SPLIT");
      return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) f = std::min(forced, 4);
  }
  int nw = 0, nc = 0, n_items = base;
  std::vector<Blk> full;
  for (const Blk& b : blks) {
    const int s = std::min(f, b.need / kMinSplitTiles);
    if (s >= 2 && nw + s <= kAttnSplitCap && n_items + s - 1 <= work_cap && nc < combine_cap) {
      mh_.combine[nc++] = make_int4(b.r, b.row0, nw, s);
      for (int k = 0; k < s; ++k)
        // .x packs the member (low 16 bits) and this block's combine entry
        // (high bits): the split CTAs find their merge ticket without a search.
        mh_.work[nw++] = make_int4(b.r | (nc - 1) << 16, b.row0, k * b.need / s, (k + 1) * b.need / s);
      n_items += s - 1;
    } else {
      full.push_back(b);
    }
  }
  for (const Blk& b : full) mh_.work[nw++] = make_int4(b.r, b.row0, 0, -1);
  mh_.scalars[2] = nw;
  mh_.scalars[3] = nc;
  }
  mh_.scalars[0] = t;
  mh_.scalars[1] = n;
  bool any_logits = false;
  for (int i = 0; i < n; ++i) any_logits = any_logits || mem[i].want_logits != 0;
  mh_.scalars[12] = any_logits ? n : 0;  // LM-head rows
  const int nw = mh_.scalars[2], nc = mh_.scalars[3];
  last_attn_pieces_ = nw;
  last_attn_merges_ = nc;
  last_attn_ctas_ = 0;
  if (attn_rows == kAttnTcRows && attn_persist_)
    for (int c = 0; c < kAttnMaxCtas; ++c) last_attn_ctas_ += mh_.cta_off[c + 1] > mh_.cta_off[c] ? 1 : 0;
  // Split-K per projection for the live token count (fused epilogues need 1).
  {
    const SplitPlan sp = plan_for(t_cap, r_cap);
    const int h = m_.hidden, D = m_.head_dim, sms = num_sms();
    const int qkv_out = (m_.n_q_heads + 2 * m_.n_kv_heads) * D;
    auto live = [&](GemmPlan gp, int M, int K, bool fused) {
      if (fused) gp.s_cap = 1;  // fused epilogues need the whole K in one unit
      return choose_tiles(M, K, gp, t, sms);
    };
    const TilePlan tq = live(sp.qkv, qkv_out, h, fuse_qkv_ && sp.qkv.splits == 1 && D == 128);
    const TilePlan to = live(sp.o, h, m_.n_q_heads * D, fuse_resid_ && sp.o.splits == 1);
    const TilePlan tg = live(sp.gu, 2 * m_.intermediate, h, true);
    const TilePlan td = live(sp.d, h, m_.intermediate, fuse_resid_ && sp.d.splits == 1);
    mh_.scalars[4] = tq.meta_splits();
    mh_.scalars[5] = to.meta_splits();
    mh_.scalars[6] = td.meta_splits();
    mh_.scalars[8] = tq.n_tiles;
    mh_.scalars[9] = to.n_tiles;
    mh_.scalars[10] = tg.n_tiles;
    mh_.scalars[11] = td.n_tiles;
  }

  last_h2d_bytes_ = 0;
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) lp_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_), "meta h2d");
    last_h2d_bytes_ += bytes;
  };
  h2d(md_.scalars, mh_.scalars, 64);
  h2d(md_.tokens, mh_.tokens, size_t(t) * 4);
  h2d(md_.positions, mh_.positions, size_t(t) * 4);
  h2d(md_.slots, mh_.slots, size_t(t) * 4);
  h2d(md_.q_start, mh_.q_start, size_t(n) * 4);
  h2d(md_.q_len, mh_.q_len, size_t(n) * 4);
  h2d(md_.hist, mh_.hist, size_t(n) * 4);
  h2d(md_.last_idx, mh_.last_idx, size_t(n) * 4);
  h2d(md_.page_off, mh_.page_off, size_t(n) * 4);
  h2d(md_.page_table, mh_.page_table, size_t(np) * 4);
  h2d(md_.work, mh_.work, size_t(nw) * 16);
  h2d(md_.combine, mh_.combine, size_t(nc) * 16);
  if (attn_rows == kAttnTcRows && attn_persist_) {
    h2d(md_.work2, mh_.work2, size_t(nw) * 16);
    h2d(md_.cta_off, mh_.cta_off, size_t(kAttnMaxCtas + 1) * 4);
  }

  lp_check(cudaEventRecord(staging_[(stage_seq_ - 1) % kStaging].h2d, stream_), "event");
  lp_check(cudaEventRecord(tk.start, stream_), "event");
  if (exec && nc == 0 && shape.kind == LP_KIND_GRAPH && !tc_graph) {
    auto it = graphs_nc_.find(graph_key(shape.l_pad, shape.depth));
    if (it != graphs_nc_.end()) exec = it->second;  // no split: skip the merge grid
  }
  {
    // Kernel count of this forward (the enqueue_forward sequence).
    const bool warp_attn = attn_rows != kAttnTcRows;
    const bool merge_grid = warp_attn && nc > 0;  // the no-merge graph variant is used when nc == 0
    const bool qkv_fused = fuse_qkv_ && plan_for(t_cap, r_cap).qkv.splits == 1 && m_.head_dim == 128;
    last_launches_ = 1 + m_.layers * (7 + (qkv_fused ? 0 : 1) + (merge_grid ? 1 : 0)) + 3;
  }
  if (exec) {
    lp_check(cudaGraphLaunch(exec, stream_), "graph launch");
  } else {
    // Standard / packed / uncaptured: eager launch sized to the live batch.
    enqueue_forward(t_cap, r_cap, stream_, false, nc > 0);
  }
  lp_check(cudaGetLastError(), "forward launch");
  lp_check(cudaEventRecord(tk.end, stream_), "event");
  // The step's result (greedy first token per member) lands in the ticket's
  // pinned slot; the host reads it once `done` fires.
  lp_check(cudaMemcpyAsync(tk.keys, next_keys_, size_t(n) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           stream_), "first tokens d2h");
  lp_check(cudaEventRecord(tk.done, stream_), "event");
  last_d2h_bytes_ = size_t(n) * sizeof(unsigned long long);
  tk.id = id;
  tk.n = n;
  tk.logits = any_logits;
  ++next_ticket_;
  for (int i = 0; i < n; ++i) {
    Session& s = sessions_[mem[i].session_id];
    s.kv_len = std::max<int64_t>(s.kv_len, mem[i].history + mem[i].new_tokens);
  }
  submitted_ = true;
  return id;
}

void Instance::timer_record(int slot) {
  if (slot < 0 || slot >= kTimerSlots) throw ShapeMismatch("timer slot out of range");
  if (!timers_[slot]) lp_check(cudaEventCreate(&timers_[slot]), "timer event");
  lp_check(cudaEventRecord(timers_[slot], stream_), "timer record");
}

double Instance::timer_elapsed(int a, int b) {
  if (a < 0 || b < 0 || a >= kTimerSlots || b >= kTimerSlots || !timers_[a] || !timers_[b])
    throw ShapeMismatch("timer slot not recorded");
  lp_check(cudaEventSynchronize(timers_[b]), "timer sync");
  float ms = 0;
  lp_check(cudaEventElapsedTime(&ms, timers_[a], timers_[b]), "timer elapsed");
  return ms;
}

double Instance::time_gemm(int layer, int which, int t_cap, int n_live, int iters) {
  if (layer < 0 || layer >= m_.layers || t_cap < 1 || t_cap > t_max_ || n_live > t_cap || iters < 1)
    throw ShapeMismatch("time_gemm: bad arguments");
  lp_check(cudaSetDevice(d_.device), "set device");
  const int h = m_.hidden, I = m_.intermediate, D = m_.head_dim;
  const int qkv_out = (m_.n_q_heads + 2 * m_.n_kv_heads) * D;
  const SplitPlan sp = plan_for(t_cap, std::min(t_cap, r_max_));
  const LayerW& w = layers_[layer];
  acquire_staging();
  GemmArgs g;
  g.N = t_cap;
  g.n_dev = md_.scalars;
  g.ws = ws_;
  g.ws_stride = t_cap;
  const CUtensorMap* tm = nullptr;
  const GemmPlan* p = nullptr;
  const bf16* x = nullptr;
  switch (which) {
    case 0: g.M = qkv_out; g.K = h; g.mode = kEpiF32Partial; tm = &w.tm_qkv; p = &sp.qkv; x = x_norm_; break;
    case 1: g.M = h; g.K = m_.n_q_heads * D; g.mode = kEpiF32Partial; tm = &w.tm_o; p = &sp.o; x = attn_; break;
    case 2: g.M = 2 * I; g.K = h; g.mode = kEpiSiluMul; g.out = act_; g.ldo = I; tm = &w.tm_gu; p = &sp.gu; x = x_norm_; break;
    case 3: g.M = h; g.K = I; g.mode = kEpiF32Partial; tm = &w.tm_d; p = &sp.d; x = act_; break;
    default: throw ShapeMismatch("time_gemm: which in 0..3");
  }
  // Same per-batch split-K choice as a forward with n_live tokens.
  mh_.scalars[0] = n_live;
  mh_.scalars[1] = std::min(n_live, r_max_);
  GemmPlan pl = *p;
  if (g.mode != kEpiF32Partial) pl.s_cap = 1;
  TilePlan tp = choose_tiles(g.M, g.K, pl, n_live, num_sms());
  if (const char* e = std::getenv("LP_TIME_GEMM_PLAN")) {  // experiments: "n_tiles,splits" (splits -1: stream-K)
    int nt = 0, s = 0;
    const int gw = gemm_workers(g.M, pl, num_sms());
    if (std::sscanf(e, "%d,%d", &nt, &s) == 2 && nt >= 1 && nt <= pl.nt_cap &&
        ((s >= 1 && s <= std::max(1, pl.s_cap)) ||
         (s == -1 && g.mode == kEpiF32Partial &&
          sk_max_segments(g.M / (128 * pl.pair), nt, g.K / 64, gw) <= pl.s_cap))) {
      tp.n_tiles = nt;
      tp.splits = std::max(1, s);
      tp.stream_k = s == -1;
    }
  }
  mh_.scalars[4] = tp.meta_splits();
  mh_.scalars[8] = tp.n_tiles;
  g.ntiles_dev = md_.scalars + 8;
  if (g.mode == kEpiF32Partial) g.splits_dev = md_.scalars + 4;
  lp_check(cudaMemcpyAsync(md_.scalars, mh_.scalars, 48, cudaMemcpyHostToDevice, stream_), "meta");
  lp_check(cudaEventRecord(staging_[(stage_seq_ - 1) % kStaging].h2d, stream_), "event");
  lp_check(cudaStreamSynchronize(stream_), "sync");
  // Realistic operand values (unit-variance activations): an all-zero input
  // would under-state power draw and over-state the clock.
  init_weights(const_cast<bf16*>(x), size_t(t_cap) * g.K, 77, 999, std::sqrt(3.0f) / 8388608.0f, 0, g.K,
               stream_);
  for (int i = 0; i < 2; ++i) gemm(*tm, *p, g, x, t_max_, stream_);  // warm-up
  lp_check(cudaEventRecord(ev_start_, stream_), "event");
  for (int i = 0; i < iters; ++i) gemm(*tm, *p, g, x, t_max_, stream_);
  lp_check(cudaEventRecord(ev_end_, stream_), "event");
  lp_check(cudaEventSynchronize(ev_end_), "sync");
  float ms = 0;
  lp_check(cudaEventElapsedTime(&ms, ev_start_, ev_end_), "elapsed");
  return ms / iters;
}

double Instance::wait() {
  if (!submitted_) throw StateError("lp_wait without a submit");
  return ticket_wait(next_ticket_ - 1);
}

void Instance::read_next_tokens(int32_t* out, int n) {
  if (!submitted_) throw StateError("lp_read_next_tokens without a submit");
  ticket_tokens(next_ticket_ - 1, out, n);
}

void Instance::read_logits(float* out, size_t cap) {
  if (!submitted_) throw StateError("lp_read_logits without a submit");
  const size_t need = size_t(ticket(next_ticket_ - 1).n) * m_.vocab;
  if (cap < need) throw ShapeMismatch("logits buffer too small");
  lp_check(cudaMemcpyAsync(out, logits_, need * 4, cudaMemcpyDeviceToHost, stream_), "d2h");
  lp_check(cudaStreamSynchronize(stream_), "d2h sync");
}

void Instance::session_pages(int64_t sid, int32_t* pages, int cap, int32_t* n_pages, int64_t* kv_len) {
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) {
    if (n_pages) *n_pages = 0;
    if (kv_len) *kv_len = 0;
    return;
  }
  const auto& s = it->second;
  if (n_pages) *n_pages = static_cast<int32_t>(s.pages.size());
  if (kv_len) *kv_len = s.kv_len;
  for (int i = 0; i < cap && i < static_cast<int>(s.pages.size()); ++i) pages[i] = s.pages[i];
}

void Instance::session_release(int64_t sid) {
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) return;
  for (int32_t p : it->second.pages) free_pages_.insert(p);
  sessions_.erase(it);
}

void Instance::read_kv(int64_t sid, int layer, int64_t pos0, int64_t n, uint16_t* k, uint16_t* v) {
  auto it = sessions_.find(sid);
  if (it == sessions_.end()) throw ShapeMismatch("unknown session");
  const Session& s = it->second;
  if (layer < 0 || layer >= m_.layers || pos0 < 0 || pos0 + n > s.kv_len)
    throw ShapeMismatch("read_kv range outside resident KV");
  lp_check(cudaStreamSynchronize(stream_), "sync");
  const int D = m_.head_dim, nkv = m_.n_kv_heads;
  std::vector<uint16_t> page(page_elems_);
  int cur = -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t pos = pos0 + i;
    const int pg = s.pages[pos / kPage];
    if (pg != cur) {
      lp_check(cudaMemcpy(page.data(), kv_pool_ + layer_stride_ * layer + size_t(pg) * page_elems_,
                          page_elems_ * 2, cudaMemcpyDeviceToHost), "kv d2h");
      cur = pg;
    }
    const int slot = static_cast<int>(pos % kPage);
    for (int g = 0; g < nkv; ++g) {
      std::memcpy(k + (i * nkv + g) * D, page.data() + (size_t(0 * nkv + g) * kPage + slot) * D, D * 2);
      std::memcpy(v + (i * nkv + g) * D, page.data() + (size_t(1 * nkv + g) * kPage + slot) * D, D * 2);
    }
  }
}

void Instance::migrate(Instance& src, Instance& dst, int64_t sid, bool keep_source) {
  auto it = src.sessions_.find(sid);
  if (it == src.sessions_.end()) return;
  if (std::memcmp(&src.m_, &dst.m_, sizeof(lp_model_desc)) != 0) throw ConfigError("model mismatch");
  dst.session_release(sid);
  Session& ss = it->second;
  Session& ds = dst.sessions_[sid];
  ds.pages = dst.alloc_pages(static_cast<int>(ss.pages.size()));
  ds.kv_len = ss.kv_len;
  const int n = static_cast<int>(ss.pages.size());
  // The source's pending forwards wrote these pages: order the copy after them.
  lp_check(cudaSetDevice(src.d_.device), "set device");
  lp_check(cudaEventRecord(src.ev_mig_, src.stream_), "src event");
  lp_check(cudaSetDevice(dst.d_.device), "set device");
  lp_check(cudaStreamWaitEvent(dst.stream_, src.ev_mig_, 0), "wait src");
  bool peer = src.d_.device == dst.d_.device;
  if (!peer) {
    int can = 0;
    cudaDeviceCanAccessPeer(&can, dst.d_.device, src.d_.device);
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(src.d_.device, 0);  // from dst's context
      if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) peer = true;
      cudaGetLastError();  // clear a benign already-enabled error
    }
  }
  if (peer) {
    // One kernel on the destination: reads the source pool directly (same
    // HBM, or the peer's HBM over NVLink) and writes the new pages.
    // Page ids travel through the destination's pinned staging buffer; the
    // previous incoming migration's H2D must have read it first.
    if (dst.mig_pending_) lp_check(cudaEventSynchronize(dst.ev_mig_done_), "migration staging reuse");
    int* h = dst.mig_host_;
    for (int k = 0; k < n; ++k) {
      h[k] = ss.pages[k];
      h[n + k] = ds.pages[k];
    }
    int* ids = dst.mig_ids_;
    lp_check(cudaMemcpyAsync(ids, h, size_t(2) * n * sizeof(int), cudaMemcpyHostToDevice, dst.stream_), "ids h2d");
    kv_page_copy(src.kv_pool_, src.layer_stride_, dst.kv_pool_, dst.layer_stride_, src.page_elems_, ids, ids + n, n,
                 src.m_.layers, dst.stream_);
    lp_check(cudaGetLastError(), "kv copy");
  } else {
    const size_t bytes = src.page_elems_ * 2;
    for (int l = 0; l < src.m_.layers; ++l) {
      for (int k = 0; k < n; ++k) {
        const bf16* from = src.kv_pool_ + src.layer_stride_ * l + size_t(ss.pages[k]) * src.page_elems_;
        bf16* to = dst.kv_pool_ + dst.layer_stride_ * l + size_t(ds.pages[k]) * dst.page_elems_;
        lp_check(cudaMemcpyPeerAsync(to, dst.d_.device, from, src.d_.device, bytes, dst.stream_), "kv p2p");
      }
    }
  }
  // No host sync: the destination's next forwards are stream-ordered after
  // the copy, and the source's stream waits for it before any later work of
  // its own can reuse the released pages.
  lp_check(cudaEventRecord(dst.ev_mig_done_, dst.stream_), "copy event");
  dst.mig_pending_ = true;
  lp_check(cudaSetDevice(src.d_.device), "set device");
  lp_check(cudaStreamWaitEvent(src.stream_, dst.ev_mig_done_, 0), "src waits for copy");
  if (!keep_source) src.session_release(sid);
}

}  // namespace lp

// ------------------------------------------------------------------ C ABI
using lp::Instance;

struct lp_instance {
  Instance* impl;
};

namespace {
// Every entry point that takes a handle validates it: a null handle is an
// LP_ERR_CONFIG status, never a crash.
Instance& impl_of(lp_instance* inst) {
  if (!inst || !inst->impl) throw lp::ConfigError("null instance handle");
  return *inst->impl;
}
}  // namespace

extern "C" {

int lp_instance_create(const lp_model_desc* model, const lp_instance_desc* desc, lp_instance** out) {
  return lp::lp_guard([&] {
    if (!model || !desc || !out) throw lp::ConfigError("null argument");
    *out = nullptr;
    auto* h = new lp_instance{nullptr};
    try {
      h->impl = new Instance(*model, *desc);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int lp_instance_destroy(lp_instance* inst) {
  return lp::lp_guard([&] {
    if (!inst) return;
    delete inst->impl;
    delete inst;
  });
}

int lp_instance_model(lp_instance* inst, lp_model_desc* out) {
  return lp::lp_guard([&] {
    if (!inst || !out) throw lp::ConfigError("null argument");
    *out = impl_of(inst).model();
  });
}

int lp_capture_graphs(lp_instance* inst, const int64_t* lengths, int32_t n_lengths, const int32_t* depths,
                      int32_t n_depths) {
  return lp::lp_guard([&] {
    if (n_lengths > 0 && !lengths) throw lp::ConfigError("null argument");
    if (n_depths > 0 && !depths) throw lp::ConfigError("null argument");
    impl_of(inst).capture_graphs(std::vector<int64_t>(lengths, lengths + n_lengths),
                               std::vector<int32_t>(depths, depths + n_depths));
  });
}

int lp_submit(lp_instance* inst, const lp_shape* shape, const lp_member* members, int32_t n,
              const int32_t* token_ids) {
  return lp::lp_guard([&] {
    if (!shape || !members || !token_ids) throw lp::ConfigError("null argument");
    impl_of(inst).submit(*shape, members, n, token_ids);
  });
}

int lp_submit_async(lp_instance* inst, const lp_shape* shape, const lp_member* members, int32_t n,
                    const int32_t* token_ids, int64_t* ticket) {
  return lp::lp_guard([&] {
    if (!shape || !members || !token_ids || !ticket) throw lp::ConfigError("null argument");
    *ticket = -1;
    *ticket = impl_of(inst).submit(*shape, members, n, token_ids);
  });
}

int lp_ticket_query(lp_instance* inst, int64_t ticket, int32_t* done) {
  return lp::lp_guard([&] {
    if (!done) throw lp::ConfigError("null argument");
    *done = impl_of(inst).ticket_done(ticket) ? 1 : 0;
  });
}

int lp_ticket_wait(lp_instance* inst, int64_t ticket, double* service_ms) {
  return lp::lp_guard([&] {
    const double ms = impl_of(inst).ticket_wait(ticket);
    if (service_ms) *service_ms = ms;
  });
}

int lp_ticket_tokens(lp_instance* inst, int64_t ticket, int32_t* out, int32_t n) {
  return lp::lp_guard([&] {
    if (!out && n > 0) throw lp::ConfigError("null argument");
    impl_of(inst).ticket_tokens(ticket, out, n);
  });
}

int lp_last_io(lp_instance* inst, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  return lp::lp_guard([&] {
    if (h2d_bytes) *h2d_bytes = static_cast<int64_t>(impl_of(inst).last_h2d_bytes_);
    if (d2h_bytes) *d2h_bytes = static_cast<int64_t>(impl_of(inst).last_d2h_bytes_);
  });
}

int lp_last_launches(lp_instance* inst, int32_t* kernels) {
  return lp::lp_guard([&] {
    if (kernels) *kernels = impl_of(inst).last_launches_;
  });
}

int lp_timer_record(lp_instance* inst, int32_t slot) {
  return lp::lp_guard([&] { impl_of(inst).timer_record(slot); });
}

int lp_timer_elapsed(lp_instance* inst, int32_t slot_a, int32_t slot_b, double* ms) {
  return lp::lp_guard([&] {
    if (!ms) throw lp::ConfigError("null argument");
    *ms = impl_of(inst).timer_elapsed(slot_a, slot_b);
  });
}

int lpk_plan_gemm(int32_t M, int32_t K, int32_t t_cap, int32_t n_live, int32_t sms, int32_t allow_split,
                  int32_t* bn, int32_t* pair, int32_t* n_tiles, int32_t* splits) {
  return lp::lp_guard([&] {
    if (M < 128 || K < 64 || t_cap < 1 || n_live < 0 || n_live > t_cap || sms < 2) throw lp::ConfigError("bad arguments");
    const lp::GemmPlan p = lp::plan_gemm_for_tests(M, K, t_cap, allow_split != 0, sms);
    lp::GemmPlan q = p;
    if (!allow_split) q.s_cap = 1;
    const lp::TilePlan t = lp::choose_tiles(M, K, q, std::max(1, n_live), sms);
    if (bn) *bn = p.bn;
    if (pair) *pair = p.pair;
    if (n_tiles) *n_tiles = t.n_tiles;
    if (splits) *splits = t.meta_splits();  // -1: stream-K
  });
}

int lpk_last_attention_schedule(lp_instance* inst, int32_t* pieces, int32_t* merges, int32_t* ctas) {
  return lp::lp_guard([&] {
    Instance& in = impl_of(inst);
    if (pieces) *pieces = in.last_attn_pieces_;
    if (merges) *merges = in.last_attn_merges_;
    if (ctas) *ctas = in.last_attn_ctas_;
  });
}

int lpk_time_gemm(lp_instance* inst, int32_t layer, int32_t which, int32_t t_cap, int32_t n_live,
                  int32_t iters, double* avg_ms) {
  return lp::lp_guard([&] {
    if (!avg_ms) throw lp::ConfigError("null argument");
    *avg_ms = impl_of(inst).time_gemm(layer, which, t_cap, n_live, iters);
  });
}

int lp_wait(lp_instance* inst, double* service_ms) {
  return lp::lp_guard([&] {
    const double ms = impl_of(inst).wait();
    if (service_ms) *service_ms = ms;
  });
}

int lp_read_next_tokens(lp_instance* inst, int32_t* out, int32_t n) {
  return lp::lp_guard([&] {
    if (!out && n > 0) throw lp::ConfigError("null argument");
    impl_of(inst).read_next_tokens(out, n);
  });
}

int lp_read_logits(lp_instance* inst, float* out, size_t cap_floats) {
  return lp::lp_guard([&] {
    if (!out) throw lp::ConfigError("null argument");
    impl_of(inst).read_logits(out, cap_floats);
  });
}

int lp_session_pages(lp_instance* inst, int64_t session_id, int32_t* pages, int32_t cap, int32_t* n_pages,
                     int64_t* kv_len) {
  return lp::lp_guard([&] { impl_of(inst).session_pages(session_id, pages, cap, n_pages, kv_len); });
}

int lp_session_release(lp_instance* inst, int64_t session_id) {
  return lp::lp_guard([&] { impl_of(inst).session_release(session_id); });
}

int lp_read_kv(lp_instance* inst, int64_t session_id, int32_t layer, int64_t pos0, int64_t n, uint16_t* k_out,
               uint16_t* v_out) {
  return lp::lp_guard([&] {
    if (!k_out || !v_out) throw lp::ConfigError("null argument");
    impl_of(inst).read_kv(session_id, layer, pos0, n, k_out, v_out);
  });
}

int lp_session_migrate(lp_instance* src, lp_instance* dst, int64_t session_id) {
  return lp::lp_guard([&] {
    Instance& a = impl_of(src);
    Instance& b = impl_of(dst);
    if (&a == &b) throw lp::ConfigError("lp_session_migrate: source and destination are the same instance");
    Instance::migrate(a, b, session_id, false);
  });
}

int lp_session_copy(lp_instance* src, lp_instance* dst, int64_t session_id) {
  return lp::lp_guard([&] {
    Instance& a = impl_of(src);
    Instance& b = impl_of(dst);
    if (&a == &b) throw lp::ConfigError("lp_session_copy: source and destination are the same instance");
    Instance::migrate(a, b, session_id, true);
  });
}

}  // extern "C"
