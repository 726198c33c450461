// Host-side schedule of the persistent tcgen05 attention (attn_tc.cu,
// attn_tcp_kernel): which (row block, kv head, page range) pieces each CTA
// walks. Pure C++ (no CUDA types), so the CPU tests drive it through
// lpk_plan_attention (laps_prefill_testing.h).
#pragma once
#include <cstddef>
#include <vector>

namespace lp {

struct AttnBlock {  // one 128-row block of a member: its causal key range is pages [0, need)
  int r, row0, need;
};
struct AttnPiece {
  int r, row0, t_begin, t_end;  // member, first row, page range
  int g;                        // kv head
  int ci;                       // combine entry of a split unit, -1 for a whole unit
  int slot;                     // fp32 partial slot (split units)
  int cta;                      // list (CTA) that runs it
};
struct AttnMerge {
  int r, row0, g, first_slot, n_pieces;
};
struct AttnSchedule {
  std::vector<AttnPiece> pieces;  // in creation order (a CTA runs its pieces in this order)
  std::vector<AttnMerge> merges;
  bool split = false;             // McNaughton lists (else whole units, longest first)
  double cap = 0, lpt_span = 0;   // list capacity / whole-unit makespan, in steps
};

// Cost model: one step per 128 keys (2 pages) + kAttnPieceCost per piece.
constexpr double kAttnPieceCost = 1.5;

// `blks` heaviest first; units = blks x nkv; `slot_cap` bounds the partial slots.
AttnSchedule plan_attention(const std::vector<AttnBlock>& blks, int nkv, int ncta, size_t slot_cap);

}  // namespace lp
