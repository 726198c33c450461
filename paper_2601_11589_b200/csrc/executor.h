// The per-GPU prefill instance behind include/laps_prefill.h.
//
// One Instance == one GPU == one reference `Inst` (sim.cpp:95-112). It owns:
//   * the random-init Qwen2-style weights (bf16, generated on device from the
//     counter-based RNG in synth.h, so the CPU oracle can regenerate them),
//   * the paged KV pool: per layer [pages][K|V][kv_head][64 slots][head_dim]
//     bf16, one page id spanning all layers, deterministic lowest-free-first
//     page allocation (restated by oracle/pages.py for bit-exact page tables),
//   * a static activation arena sized for the largest forward, shared by every
//     captured graph,
//   * per-(l_pad, depth) CUDA graphs (GraphGrid, scheduler.hpp:21-32) whose
//     kernels read live token/member counts from a device metadata block, so
//     a replay never depends on the history lengths H_i.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "../../include/laps_prefill.h"
#include "attn.cuh"
#include "gemm_sm100.cuh"
#include "ops.cuh"

namespace lp {

struct LayerW {
  bf16 *wqkv, *bqkv, *wo, *wgu, *wd, *g_attn, *g_mlp;
  CUtensorMap tm_qkv, tm_o, tm_gu, tm_d;
};

struct Session {
  std::vector<int32_t> pages;
  int64_t kv_len = 0;
};

// Device metadata block (one allocation, regions at fixed offsets).
struct Meta {
  int* scalars;     // [0] n_tokens, [1] n_members, [2] n_work
  int* tokens;      // [T]
  int* positions;   // [T]
  int* slots;       // [T]
  int* q_start;     // [R]
  int* q_len;       // [R]
  int* hist;        // [R]
  int* last_idx;    // [R]
  int* page_table;  // flattened page ids of all members (ragged)
  int* page_off;    // [R] offset of member r in page_table
  int4* work;       // [W] attention work items (see attn.cuh)
  int4* combine;    // [C] split row blocks to merge
  int4* work2;      // [W] persistent attention pieces: (kv head, combine entry, partial slot, 0)
  int* cta_off;     // [kAttnMaxCtas + 1] persistent attention: first piece of each CTA
};

// Launch plan of one projection at a given token capacity.
struct GemmPlan {
  int bn = 16;     // token tile
  int pair = 1;    // 2 = cta_group::2 CTA pair
  int splits = 1;  // split-K factor at full capacity (fp32 partial epilogues only)
  int s_cap = 1;   // largest split-K factor the workspace allows at this capacity
  int nt_cap = 1;  // largest token-tile count a per-batch tile plan may pick
};
int choose_splits(int M, int bn, int pair, int n_live, int s_cap, int sms);
struct TilePlan {
  int n_tiles = 1, splits = 1;
  bool stream_k = false;  // stream-K over the flattened (tile, K-block) space (splits unused)
  int meta_splits() const { return stream_k ? -1 : splits; }  // the device metadata value
};
TilePlan choose_tiles(int M, int K, const GemmPlan& p, int n_live, int sms);
GemmPlan plan_gemm_for_tests(int M, int K, int t_cap, bool allow_split, int sms);  // lpk_plan_gemm
struct SplitPlan {
  GemmPlan qkv, o, gu, d, lm;
};

class Instance {
 public:
  Instance(const lp_model_desc& m, const lp_instance_desc& d);
  ~Instance();

  void capture_graphs(const std::vector<int64_t>& lens, const std::vector<int32_t>& depths);
  // Asynchronous: returns the ticket id of this forward (see Ticket).
  int64_t submit(const lp_shape& shape, const lp_member* members, int n, const int32_t* tokens);
  double wait();  // the last submit
  void read_next_tokens(int32_t* out, int n);
  // Per-forward results (first tokens, device time) stay readable for the
  // last kTickets submits; an older ticket is expired (LP_ERR_STATE).
  bool ticket_done(int64_t id);
  double ticket_wait(int64_t id);
  void ticket_tokens(int64_t id, int32_t* out, int n);
  void read_logits(float* out, size_t cap);
  void session_pages(int64_t sid, int32_t* pages, int cap, int32_t* n_pages, int64_t* kv_len);
  void session_release(int64_t sid);
  void read_kv(int64_t sid, int layer, int64_t pos0, int64_t n, uint16_t* k, uint16_t* v);
  static void migrate(Instance& src, Instance& dst, int64_t sid, bool keep_source);
  void timer_record(int slot);
  double timer_elapsed(int a, int b);
  double time_gemm(int layer, int which, int t_cap, int n_live, int iters);
  static constexpr int kTimerSlots = 8;

  const lp_model_desc& model() const { return m_; }
  int device() const { return d_.device; }

 private:
  void alloc_weights();
  void alloc_arena();
  SplitPlan plan_for(int t_cap, int r_cap) const;
  void enqueue_forward(int t_cap, int r_cap, cudaStream_t st, bool graph, bool combine = true);
  const CUtensorMap& act_map(const bf16* buf, int rows, int cols, int box_rows);
  void gemm(const CUtensorMap& tm_w, const GemmPlan& p, GemmArgs g, const bf16* x, int x_rows, cudaStream_t st);
  std::vector<int32_t> alloc_pages(int n);
  void ensure_capacity(Session& s, int64_t tokens);
  int64_t graph_key(int64_t l_pad, int depth) const { return l_pad * 1024 + depth; }

  lp_model_desc m_;
  lp_instance_desc d_;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_start_ = nullptr, ev_end_ = nullptr;  // time_gemm only
  cudaEvent_t ev_mig_ = nullptr;       // end of this instance's queued work, for a session migration
  cudaEvent_t ev_mig_done_ = nullptr;  // an incoming migration's copy finished reading the ids
  bool mig_pending_ = false;

  // Host -> device metadata goes through kStaging pinned blocks used round
  // robin, so the host can prepare forward k+1..k+3 while forward k runs;
  // a block is rewritten only after its previous H2D copies drained.
  static constexpr int kStaging = 4;
  struct Staging {
    void* host = nullptr;
    Meta m{};
    cudaEvent_t h2d = nullptr;
    bool used = false;
  };
  Staging staging_[kStaging];
  int64_t stage_seq_ = 0;
  Meta& acquire_staging();  // points mh_ at the next free block
  // One slot per in-flight forward: device-time events and a pinned copy of
  // the greedy first tokens, written by a D2H at the end of the forward.
  static constexpr int kTickets = 16;
  struct Ticket {
    int64_t id = -1;
    int n = 0;
    bool logits = true;  // the forward ran the LM head (some member wanted its first token)
    cudaEvent_t start = nullptr, end = nullptr, done = nullptr;
    unsigned long long* keys = nullptr;  // pinned [r_max]
  };
  Ticket tickets_[kTickets];
  int64_t next_ticket_ = 0;
  Ticket& ticket(int64_t id);

  // model
  std::vector<LayerW> layers_;
  bf16 *embed_ = nullptr, *lm_head_ = nullptr, *g_final_ = nullptr;
  CUtensorMap tm_lm_;
  float* inv_freq_ = nullptr;
  std::vector<void*> allocs_;

  // kv
  bf16* kv_pool_ = nullptr;
  size_t layer_stride_ = 0;  // elements per layer
  size_t page_elems_ = 0;    // elements per page per layer
  int64_t n_pages_ = 0;
  std::set<int32_t> free_pages_;
  std::unordered_map<int64_t, Session> sessions_;
  int max_pages_ = 0;  // page-table row stride

  // arena
  int t_max_ = 0, r_max_ = 0, w_max_ = 0, c_max_ = 0;
  float* attn_ws_o_ = nullptr;
  float* attn_ws_ml_ = nullptr;
  int* attn_comb_cnt_ = nullptr;  // split arrival tickets: the last split CTA merges its row block
  CUtensorMap tm_kv_;
  int work_cap_for(int t_cap, int r_cap) const;
  int combine_cap_for(int t_cap, int r_cap) const;
  int block_cap_for(int t_cap, int r_cap) const;
  float* x_resid_ = nullptr;
  bf16 *x_norm_ = nullptr, *q_ = nullptr, *attn_ = nullptr, *act_ = nullptr, *x_last_ = nullptr;
  float* ws_ = nullptr;
  size_t ws_elems_ = 0;
  int* sk_tab_ = nullptr;  // stream-K segment table (GemmArgs::sk_tab)
  float* logits_ = nullptr;
  unsigned long long* next_keys_ = nullptr;
  void* meta_dev_ = nullptr;
  int* mig_ids_ = nullptr;   // device page-id lists of an incoming migration
  int* mig_host_ = nullptr;  // pinned staging for them
  size_t meta_bytes_ = 0;
  Meta md_{}, mh_{};
  std::map<std::tuple<const void*, int, int>, CUtensorMap> act_maps_;

  cudaEvent_t timers_[kTimerSlots] = {};
  // Fused GEMM epilogues (QKV bias+RoPE+KV append, residual add) for GEMMs
  // whose capacity plan has no split-K. Measured neutral against the split
  // reduction kernels, and they pin the runtime split-K to 1, so they are
  // opt-in (LP_FUSE_EPI=1); the default chooses split-K per batch.
  bool fuse_qkv_ = false, fuse_resid_ = false;
  // Graph replays of at least this many tokens use the tcgen05 attention
  // kernel (LP_GRAPH_ATTN_TC_MIN); smaller graphs the warp-MMA one.
  int graph_tc_min_ = 1 << 30;
  int attn_rows_for(bool graph, int t_cap) const {
    return (graph && t_cap < graph_tc_min_) ? kAttnRows : attn_rows_;
  }
  // head_dim 128 attention on the tcgen05/TMEM kernel (128-row work items);
  // LP_ATTN_TC=0 selects the warp-MMA kernel (64-row items) instead.
  bool attn_tc_ = true;
  int attn_rows_ = kAttnRows;
  // The tcgen05 attention runs as a persistent grid (one CTA per SM) over a
  // balanced piece schedule built per batch (LP_ATTN_PERSIST=0: one CTA per
  // work item, the round-1 launch).
  bool attn_persist_ = true;
  int pw_max_ = 0;  // persistent pieces capacity
  int plan_persistent_attention(int n, int G);

  // graphs
  std::map<int64_t, cudaGraphExec_t> graphs_;
  // Single-member standard launches (long-prefill chunks, scheduler.cpp:322-338)
  // replay graphs captured per 64-token capacity up to kChunkGraphMax
  // (= C_l, scheduler.hpp:46): an eager chunk forward is ~300 launches, which
  // the host cannot issue as fast as the GPU retires them.
  static constexpr int kChunkGraphStep = 64, kChunkGraphMax = 512;
  std::map<int, cudaGraphExec_t> chunk_graphs_;
  cudaGraphExec_t capture_one(int t_cap, int r_cap, bool graph_attn, bool combine = true);
  // Grid shapes also get a variant without the attention merge grid, replayed
  // when no row block of the batch was split (every H = 0 batch, e.g.).
  std::map<int64_t, cudaGraphExec_t> graphs_nc_;
  // ... and a variant on the tcgen05 attention kernel, replayed when the
  // batch's attention work sum_i L_i (H_i + L_i) reaches graph_tc_pairs_ with
  // >= 512 keys per query on average (deep
  // re-prefill buckets: measured 0.62 -> 0.68 of roofline at 256x4, H=1024;
  // the warp-MMA kernel stays faster for short rows).
  std::map<int64_t, cudaGraphExec_t> graphs_tc_;
  int64_t graph_tc_pairs_ = 500000;  // LP_GRAPH_TC_PAIRS overrides
  bool submitted_ = false;  // a forward was submitted (lp_wait / lp_read_next_tokens refer to it)
 public:
  size_t last_h2d_bytes_ = 0, last_d2h_bytes_ = 0;  // host<->device bytes of the last submit / read
  int last_launches_ = 0;                             // kernels of the last submit
  int last_attn_pieces_ = 0, last_attn_merges_ = 0, last_attn_ctas_ = 0;  // attention schedule of the last submit
};

}  // namespace lp
