// Decoding path generation (NEXT-1): Alg 5 (DPG) on the host, graph only.
//
// Equations: every received LT row j (Y_j = XOR_{m in N(j)} I_m, PAPER.md:91 step (2)) and every
// precode check i (0 = XOR_{m in P(i)} D_m ^ C_i, step (1)); "BP at most twice (once for the
// outer graph code and ... the inner precode)" becomes one peeling over the union
// of both equation sets.  Level L (Alg 5's iteration i): the equations with exactly one unknown
// left given the symbols recovered at levels < L; each such unknown is recovered by ONE of them,
// the lowest-degree one (ties: the lowest equation index, LT rows before checks),
// so a level's rows are independent (no intra-level dependency).  The recovered set
// at convergence equals Alg 1's: the complement of the largest stopping set.
#include <algorithm>

#include "fsb_internal.h"

namespace fsb {

fs_status build_decode_plan(const Graph &g, const uint8_t *received, DecodePlan &pl) {
  const uint32_t k = g.prm.k, p = g.prm.p, n = g.prm.n, K = k + p;
  pl = DecodePlan();
  pl.k = k, pl.p = p, pl.n = n, pl.K = K, pl.t = g.prm.t;
  // equations 0..n-1: LT rows (only received ones are used); n..n+p-1: precode checks
  const uint32_t E = n + p;
  std::vector<uint32_t> deg(E, 0), unknown(E, 0);
  std::vector<uint8_t> active(E, 0);
  auto members = [&](uint32_t e, auto &&fn) {
    if (e < n) {
      for (int32_t x = g.lt_row_ptr[e]; x < g.lt_row_ptr[e + 1]; ++x) fn(static_cast<uint32_t>(g.lt_col[x]));
    } else {
      const uint32_t i = e - n;
      for (int32_t x = g.pre_row_ptr[i]; x < g.pre_row_ptr[i + 1]; ++x) fn(static_cast<uint32_t>(g.pre_col[x]));
      fn(k + i);
    }
  };
  // symbol -> equations (transpose)
  std::vector<uint32_t> sym_ptr(K + 1, 0);
  for (uint32_t e = 0; e < E; ++e) {
    active[e] = e < n ? (received[e] ? 1 : 0) : 1;
    if (e < n && received[e]) ++pl.received;
    if (!active[e]) continue;
    members(e, [&](uint32_t m) { ++sym_ptr[m + 1]; ++deg[e]; });
    unknown[e] = deg[e];
  }
  for (uint32_t m = 0; m < K; ++m) sym_ptr[m + 1] += sym_ptr[m];
  std::vector<uint32_t> sym_eq(sym_ptr[K]);
  {
    std::vector<uint32_t> fill(sym_ptr.begin(), sym_ptr.end() - 1);
    for (uint32_t e = 0; e < E; ++e)
      if (active[e]) members(e, [&](uint32_t m) { sym_eq[fill[m]++] = e; });
  }
  pl.state.assign(K, 0);
  pl.level_of.assign(K, -1);
  pl.level_ptr.assign(1, 0);
  pl.src_ptr.assign(1, 0);
  std::vector<uint32_t> cand;
  for (uint32_t e = 0; e < E; ++e)
    if (active[e] && unknown[e] == 1) cand.push_back(e);
  std::vector<uint32_t> chosen_eq(K, UINT32_MAX);
  std::vector<uint32_t> level_syms;
  while (!cand.empty()) {
    const int32_t L = static_cast<int32_t>(pl.level_ptr.size()) - 1;
    // each candidate's single unknown; keep the lowest-degree equation per unknown
    level_syms.clear();
    for (uint32_t e : cand) {
      if (unknown[e] != 1) continue;
      uint32_t f = UINT32_MAX;
      members(e, [&](uint32_t m) {
        if (!pl.state[m]) f = m;
      });
      if (f == UINT32_MAX) continue;
      if (chosen_eq[f] == UINT32_MAX) {
        chosen_eq[f] = e;
        level_syms.push_back(f);
      } else if (deg[e] < deg[chosen_eq[f]] || (deg[e] == deg[chosen_eq[f]] && e < chosen_eq[f])) {
        chosen_eq[f] = e;
      }
    }
    if (level_syms.empty()) break;
    std::sort(level_syms.begin(), level_syms.end());
    for (uint32_t f : level_syms) {
      const uint32_t e = chosen_eq[f];
      pl.target.push_back(static_cast<int32_t>(f));
      if (e < n) pl.src.push_back(e | kSrcCoded);  // rhs: received coded row e
      members(e, [&](uint32_t m) {
        if (m != f) pl.src.push_back(m);
      });
      pl.src.back() |= kSrcLast;
      pl.src_ptr.push_back(static_cast<int32_t>(pl.src.size()));
    }
    pl.level_ptr.push_back(static_cast<uint32_t>(pl.target.size()));
    // mark the level's symbols recovered, then update the equations' unknown counts
    std::vector<uint32_t> next;
    for (uint32_t f : level_syms) {
      pl.state[f] = 1;
      pl.level_of[f] = L;
    }
    for (uint32_t f : level_syms)
      for (uint32_t x = sym_ptr[f]; x < sym_ptr[f + 1]; ++x) {
        const uint32_t e = sym_eq[x];
        if (--unknown[e] == 1) next.push_back(e);
      }
    std::sort(next.begin(), next.end());
    next.erase(std::unique(next.begin(), next.end()), next.end());
    cand.swap(next);
  }
  return FS_OK;
}

}  // namespace fsb
