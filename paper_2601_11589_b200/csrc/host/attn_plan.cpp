// Balanced piece lists for the persistent tcgen05 attention (attn_plan.h).
//
// A unit = (128-row block, kv head) over the block's causal key range. The
// units, heaviest first, are cut into ncta lists of equal cost with
// McNaughton's wrap-around rule — units are divisible along the keys, so a
// unit crossing a list boundary becomes pieces whose fp32 partials the
// last-finishing piece merges — at the smallest capacity (bisection) that
// does not overload the last list. That split schedule pays more than its
// nominal per-piece cost (merge, partial round trip, a cold pipeline), so it
// is used only when it beats whole units placed longest-first on the
// least-loaded list by 15 % + 6 steps (measured on 7B / 32B chunks at
// H = 0..16 K, profiles/r02_attn_experiments.md).
#include "../attn_plan.h"

#include <algorithm>

namespace lp {

namespace {

int steps_of(int pages) { return (pages + 1) / 2; }

// One walk at list capacity `cap`; returns the load of the last list.
double walk(const std::vector<AttnBlock>& blks, int nkv, int ncta, size_t slot_cap, double cap,
            AttnSchedule* out) {
  int cta = 0, slots = 0, merges = 0;
  double load = 0;
  for (const AttnBlock& b : blks) {
    for (int g = 0; g < nkv; ++g) {
      int p0 = 0, pieces = 0;
      const size_t first = out ? out->pieces.size() : 0;
      while (p0 < b.need) {
        const int rem = steps_of(b.need - p0);
        const double room = cap - load - kAttnPieceCost;
        const int take = room > 0 ? static_cast<int>(room) : 0;
        if (cta == ncta - 1 || rem <= room + 0.5) {  // the rest fits (or this is the last list)
          if (out) out->pieces.push_back(AttnPiece{b.r, b.row0, p0, b.need, g, -1, 0, cta});
          ++pieces;
          load += rem + kAttnPieceCost;
          p0 = b.need;
        } else {
          if (take >= 1 && rem - take >= 1 && size_t(slots + pieces) + 2 <= slot_cap) {
            if (out) out->pieces.push_back(AttnPiece{b.r, b.row0, p0, p0 + 2 * take, g, -1, 0, cta});
            ++pieces;
            p0 += 2 * take;
          }
          ++cta;
          load = 0;
        }
        if (load >= cap - 1e-9 && cta < ncta - 1) {
          ++cta;
          load = 0;
        }
      }
      if (pieces > 1) {
        if (out) {
          for (int k = 0; k < pieces; ++k) {
            AttnPiece& pc = out->pieces[first + static_cast<size_t>(k)];
            pc.ci = merges;
            pc.slot = slots + k;
          }
          out->merges.push_back(AttnMerge{b.r, b.row0, g, slots, pieces});
        }
        ++merges;
        slots += pieces;
      }
    }
  }
  return cta == ncta - 1 ? load : 0.0;
}

}  // namespace

AttnSchedule plan_attention(const std::vector<AttnBlock>& blks, int nkv, int ncta, size_t slot_cap) {
  AttnSchedule s;
  double total = 0, biggest = 0;
  for (const AttnBlock& b : blks) {
    const double cost = steps_of(b.need) + kAttnPieceCost;
    total += nkv * cost;
    biggest = std::max(biggest, cost);
  }
  double lo = total / ncta, hi = lo + 2 * biggest;
  for (int it = 0; it < 24 && hi - lo > 0.25; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (walk(blks, nkv, ncta, slot_cap, mid, nullptr) <= mid + 0.5) hi = mid;
    else lo = mid;
  }
  // Whole units, longest first, each onto the least-loaded list.
  std::vector<double> load(static_cast<size_t>(ncta), 0.0);
  std::vector<int> list_of;
  for (const AttnBlock& b : blks) {
    for (int g = 0; g < nkv; ++g) {
      const size_t c = static_cast<size_t>(std::min_element(load.begin(), load.end()) - load.begin());
      load[c] += steps_of(b.need) + kAttnPieceCost;
      list_of.push_back(static_cast<int>(c));
    }
  }
  s.cap = hi;
  s.lpt_span = *std::max_element(load.begin(), load.end());
  s.split = 1.15 * hi + 6.0 < s.lpt_span;
  if (s.split) {
    walk(blks, nkv, ncta, slot_cap, hi, &s);
  } else {
    size_t u = 0;
    for (const AttnBlock& b : blks)
      for (int g = 0; g < nkv; ++g, ++u) s.pieces.push_back(AttnPiece{b.r, b.row0, 0, b.need, g, -1, 0, list_of[u]});
  }
  return s;
}

}  // namespace lp

// ---- test hook (laps_prefill_testing.h)
#include "../abi_common.h"

extern "C" int lpk_plan_attention(const int32_t* needs, int32_t n_blocks, int32_t nkv, int32_t ncta,
                                  int32_t* out, int32_t cap, int32_t* n_pieces, int32_t* n_merges,
                                  double* list_cap, double* lpt_span) {
  return lp::lp_guard([&] {
    if (!needs || n_blocks < 0 || nkv < 1 || ncta < 1 || !n_pieces) throw lp::ConfigError("bad arguments");
    std::vector<lp::AttnBlock> blks;
    for (int i = 0; i < n_blocks; ++i) blks.push_back(lp::AttnBlock{0, i, needs[i]});
    const lp::AttnSchedule s = lp::plan_attention(blks, nkv, ncta, size_t(1024) * nkv);
    *n_pieces = static_cast<int32_t>(s.pieces.size());
    if (n_merges) *n_merges = static_cast<int32_t>(s.merges.size());
    if (list_cap) *list_cap = s.cap;
    if (lpt_span) *lpt_span = s.split ? -1.0 : s.lpt_span;
    if (!out) return;
    if (static_cast<int32_t>(s.pieces.size()) > cap) throw lp::ShapeMismatch("output capacity too small");
    for (size_t k = 0; k < s.pieces.size(); ++k) {
      const lp::AttnPiece& p = s.pieces[k];
      int32_t* o = out + 6 * k;
      o[0] = p.cta;
      o[1] = p.row0;  // block index
      o[2] = p.g;
      o[3] = p.t_begin;
      o[4] = p.t_end;
      o[5] = p.ci;
    }
  });
}
