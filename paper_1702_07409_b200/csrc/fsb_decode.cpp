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

namespace {

// Equation e's members: LT row e (e < n) or precode check e-n with its check symbol k+(e-n).
struct Members {
  const Graph &g;
  template <typename F>
  void operator()(uint32_t e, F &&fn) const {
    const uint32_t n = g.prm.n, k = g.prm.k;
    if (e < n) {
      for (int32_t x = g.lt_row_ptr[e]; x < g.lt_row_ptr[e + 1]; ++x) fn(static_cast<uint32_t>(g.lt_col[x]));
    } else {
      const uint32_t i = e - n;
      for (int32_t x = g.pre_row_ptr[i]; x < g.pre_row_ptr[i + 1]; ++x) fn(static_cast<uint32_t>(g.pre_col[x]));
      fn(k + i);
    }
  }
};
Members members_fn(const Graph &g) { return Members{g}; }

// Completing the decode after peeling stalls ("needs an inactivation /
// GF(2) fallback at these overheads"; not in the paper, whose decoder is BP only): inactivation
// decoding.  While unknowns remain, peel any equation with one unresolved member; when none has,
// *inactivate* an unknown (the one in the most two-unknown equations, ties: lowest index) and
// carry it symbolically.  A symbol peeled in this phase gets a partial value P_x = its equation's
// right-hand side XOR its other non-inactivated members (rows of the intermediate buffer), with
// P_x = I_x XOR (XOR of the inactivated symbols in its dependence set D_x).  Every equation not
// used for peeling (the leftover) gives Z_k = Y_k XOR its non-inactivated members (a workspace
// row) = XOR of the inactivated symbols in c_k.  Gauss-Jordan on the c_k (augmented with the
// leftover index) decides, for each inactivated j (vector e_j) and each peeled x (vector D_x),
// whether it lies in the row space -- exactly the symbols the received equations determine --
// and as which XOR of Z rows; the final level writes I_j = XOR Z, I_x = P_x XOR Z (in place).
// Levels: dependencies as in the peeling; all final rows in one last level.
fs_status inactivation_phase(const Graph &g, const uint8_t *received, DecodePlan &pl, const Members &members,
                             const std::vector<uint32_t> &chosen_eq) {
  const uint32_t n = g.prm.n, p = g.prm.p, K = g.prm.k + p, E = n + p;
  std::vector<uint8_t> used(E, 0), active(E, 0);
  for (uint32_t m = 0; m < K; ++m)
    if (pl.state[m] && chosen_eq[m] != UINT32_MAX) used[chosen_eq[m]] = 1;
  for (uint32_t e = 0; e < E; ++e) active[e] = e < n ? (received[e] ? 1 : 0) : 1;
  // resolved = peeled (DPG or this phase) or inactivated
  std::vector<uint8_t> resolved(pl.state.begin(), pl.state.end());
  uint32_t nunres = 0;
  for (uint32_t m = 0; m < K; ++m) nunres += resolved[m] ? 0 : 1;
  if (!nunres) return FS_OK;
  std::vector<uint32_t> unres(E, 0);
  std::vector<uint32_t> sym_ptr(K + 1, 0);
  for (uint32_t e = 0; e < E; ++e)
    if (active[e]) members(e, [&](uint32_t m) { ++sym_ptr[m + 1]; });
  for (uint32_t m = 0; m < K; ++m) sym_ptr[m + 1] += sym_ptr[m];
  std::vector<uint32_t> sym_eq(sym_ptr[K]);
  {
    std::vector<uint32_t> fill(sym_ptr.begin(), sym_ptr.end() - 1);
    for (uint32_t e = 0; e < E; ++e)
      if (active[e])
        members(e, [&](uint32_t m) {
          sym_eq[fill[m]++] = e;
          if (!resolved[m]) ++unres[e];
        });
  }
  // symbol kinds: 0 DPG-peeled (final value), 1 peeled here (partial value), 2 inactivated,
  // 3 in no received equation at all (cannot be determined; nothing to carry)
  std::vector<uint8_t> kind(K, 0);
  std::vector<int32_t> inact_of(K, -1);  // column of an inactivated symbol
  std::vector<uint32_t> inact;
  std::vector<std::vector<uint64_t>> D(K);  // dependence sets of kind-1 symbols (bitsets)
  auto xor_into = [](std::vector<uint64_t> &a, const std::vector<uint64_t> &b) {
    if (a.size() < b.size()) a.resize(b.size(), 0);
    for (size_t w = 0; w < b.size(); ++w) a[w] ^= b[w];
  };
  auto level_of_src = [&](uint32_t m) { return pl.level_of[m]; };
  std::vector<uint32_t> q;  // equations that may have one unresolved member
  for (uint32_t e = 0; e < E; ++e)
    if (active[e] && !used[e] && unres[e] == 1) q.push_back(e);
  std::vector<std::pair<uint32_t, uint32_t>> phase_rows;  // (symbol, equation) in peel order
  for (uint32_t m = 0; m < K; ++m)
    if (!resolved[m] && sym_ptr[m + 1] == sym_ptr[m]) kind[m] = 3, resolved[m] = 1, --nunres;
  auto resolve = [&](uint32_t x) {
    resolved[x] = 1;
    --nunres;
    for (uint32_t y = sym_ptr[x]; y < sym_ptr[x + 1]; ++y) {
      const uint32_t e = sym_eq[y];
      if (--unres[e] == 1 && !used[e]) q.push_back(e);
    }
  };
  size_t qh = 0;
  while (nunres) {
    if (qh < q.size()) {
      const uint32_t e = q[qh++];
      if (used[e] || unres[e] != 1) continue;
      uint32_t x = UINT32_MAX;
      members(e, [&](uint32_t m) {
        if (!resolved[m]) x = m;
      });
      used[e] = 1;
      kind[x] = 1;
      std::vector<uint64_t> d;
      members(e, [&](uint32_t m) {
        if (m == x) return;
        if (kind[m] == 2) {
          const uint32_t c = static_cast<uint32_t>(inact_of[m]);
          if (d.size() <= c / 64) d.resize(c / 64 + 1, 0);
          d[c / 64] ^= 1ull << (c % 64);
        } else if (kind[m] == 1) {
          xor_into(d, D[m]);
        }
      });
      D[x].swap(d);
      phase_rows.push_back({x, e});
      resolve(x);
      continue;
    }
    // stuck: inactivate the unresolved symbol in the most two-unknown equations
    std::vector<uint32_t> cnt(K, 0);
    uint32_t best = UINT32_MAX;
    for (uint32_t e = 0; e < E; ++e) {
      if (!active[e] || used[e] || unres[e] != 2) continue;
      members(e, [&](uint32_t m) {
        if (!resolved[m]) ++cnt[m];
      });
    }
    for (uint32_t m = 0; m < K; ++m)
      if (!resolved[m] && (best == UINT32_MAX || cnt[m] > cnt[best])) best = m;
    kind[best] = 2;
    inact_of[best] = static_cast<int32_t>(inact.size());
    inact.push_back(best);
    resolve(best);
  }
  // rows of the peeled-here symbols (partial values) in dependency levels after the DPG levels
  const int32_t L0 = static_cast<int32_t>(pl.level_ptr.size()) - 1;  // first new level
  struct Row {
    int32_t target;           // symbol, or workspace row | kSrcWork
    std::vector<uint32_t> src;
    int32_t level;
  };
  std::vector<Row> rows;
  std::vector<int32_t> wlevel;  // level of each workspace row
  for (auto [x, e] : phase_rows) {
    Row r{static_cast<int32_t>(x), {}, L0};
    int32_t lv = L0;
    if (e < n) r.src.push_back(e | kSrcCoded);
    members(e, [&](uint32_t m) {
      if (m == x || kind[m] == 2) return;
      r.src.push_back(m);
      lv = std::max(lv, level_of_src(m) + 1);
    });
    r.level = lv;
    pl.level_of[x] = lv;  // provisional (partial value), for the dependants' levels
    rows.push_back(std::move(r));
  }
  // leftover equations: c_k over the inactivated symbols.  Only a basis of them is needed (at
  // most one per inactivated symbol): an equation whose c_k is independent of the ones kept so far
  // is kept, and its Z_k computed into a workspace row.
  const uint32_t ni = static_cast<uint32_t>(inact.size());
  const uint32_t Wi = (ni + 63) / 64;
  std::vector<std::vector<uint64_t>> C;
  std::vector<uint32_t> zrow_eq;
  std::vector<std::vector<uint64_t>> basis;  // reduced copies, basis[b] has pivot bpiv[b]
  std::vector<uint32_t> bpiv;
  for (uint32_t e = 0; e < E && C.size() < ni; ++e) {
    if (!active[e] || used[e]) continue;
    std::vector<uint64_t> c(Wi, 0);
    members(e, [&](uint32_t m) {
      if (kind[m] == 2) c[inact_of[m] / 64] ^= 1ull << (inact_of[m] % 64);
      else if (kind[m] == 1) xor_into(c, D[m]);
    });
    c.resize(Wi);
    std::vector<uint64_t> red = c;
    for (size_t b = 0; b < basis.size(); ++b)
      if (red[bpiv[b] / 64] & (1ull << (bpiv[b] % 64)))
        for (uint32_t w = 0; w < Wi; ++w) red[w] ^= basis[b][w];
    uint32_t pv = UINT32_MAX;
    for (uint32_t w = 0; w < Wi && pv == UINT32_MAX; ++w)
      if (red[w]) pv = w * 64 + static_cast<uint32_t>(__builtin_ctzll(red[w]));
    if (pv == UINT32_MAX) continue;  // dependent on the kept ones (or 0 = 0): no new information
    basis.push_back(std::move(red));
    bpiv.push_back(pv);
    const uint32_t wk = static_cast<uint32_t>(zrow_eq.size());
    Row r{static_cast<int32_t>(wk | kSrcWork), {}, L0};
    int32_t lv = L0;
    if (e < n) r.src.push_back(e | kSrcCoded);
    members(e, [&](uint32_t m) {
      if (kind[m] == 2) return;
      r.src.push_back(m);
      lv = std::max(lv, level_of_src(m) + 1);
    });
    r.level = lv;
    wlevel.push_back(lv);
    rows.push_back(std::move(r));
    C.push_back(std::move(c));
    zrow_eq.push_back(e);
  }
  // Gauss-Jordan on C augmented with the identity over the Z rows
  const uint32_t nz = static_cast<uint32_t>(C.size()), Wz = (nz + 63) / 64, W = Wi + Wz;
  std::vector<uint64_t> M(static_cast<size_t>(nz) * W, 0);
  for (uint32_t r = 0; r < nz; ++r) {
    std::copy(C[r].begin(), C[r].end(), M.begin() + static_cast<size_t>(r) * W);
    M[static_cast<size_t>(r) * W + Wi + r / 64] |= 1ull << (r % 64);
  }
  std::vector<int32_t> pivcol;
  uint32_t piv = 0;
  for (uint32_t c = 0; c < ni && piv < nz; ++c) {
    const uint32_t w = c / 64;
    const uint64_t bit = 1ull << (c % 64);
    uint32_t r = piv;
    while (r < nz && !(M[static_cast<size_t>(r) * W + w] & bit)) ++r;
    if (r == nz) continue;
    if (r != piv)
      std::swap_ranges(M.begin() + static_cast<size_t>(r) * W, M.begin() + static_cast<size_t>(r + 1) * W,
                       M.begin() + static_cast<size_t>(piv) * W);
    const uint64_t *pr = &M[static_cast<size_t>(piv) * W];
    for (uint32_t o = 0; o < nz; ++o) {
      if (o == piv) continue;
      uint64_t *ro = &M[static_cast<size_t>(o) * W];
      if (ro[w] & bit)
        for (uint32_t x = w; x < W; ++x) ro[x] ^= pr[x];
    }
    pivcol.push_back(static_cast<int32_t>(c));
    ++piv;
  }
  // reduce a vector over the inactivated symbols; true (and the Z set) if it is in the row space
  auto express = [&](std::vector<uint64_t> v, std::vector<uint64_t> &zset) {
    v.resize(Wi, 0);
    zset.assign(Wz, 0);
    for (uint32_t r = 0; r < piv; ++r) {
      const uint32_t c = static_cast<uint32_t>(pivcol[r]);
      if (!(v[c / 64] & (1ull << (c % 64)))) continue;
      const uint64_t *row = &M[static_cast<size_t>(r) * W];
      for (uint32_t x = 0; x < Wi; ++x) v[x] ^= row[x];
      for (uint32_t x = 0; x < Wz; ++x) zset[x] ^= row[Wi + x];
    }
    for (uint64_t w : v)
      if (w) return false;
    return true;
  };
  int32_t maxL = L0;
  for (const Row &r : rows) maxL = std::max(maxL, r.level);
  const int32_t Lf = maxL + 1;  // the final level, after every partial value and Z row
  std::vector<uint64_t> zset;
  auto final_row = [&](uint32_t x, bool in_place) {
    Row r{static_cast<int32_t>(x), {}, Lf};
    if (in_place) r.src.push_back(x);
    for (uint32_t w = 0; w < Wz; ++w)
      for (uint64_t bits = zset[w]; bits; bits &= bits - 1)
        r.src.push_back((w * 64 + static_cast<uint32_t>(__builtin_ctzll(bits))) | kSrcWork);
    rows.push_back(std::move(r));
    pl.state[x] = 2;
  };
  for (uint32_t j = 0; j < ni; ++j) {
    std::vector<uint64_t> v(Wi, 0);
    v[j / 64] |= 1ull << (j % 64);
    if (express(v, zset)) final_row(inact[j], false);
  }
  for (auto [x, e] : phase_rows) {
    (void)e;
    bool empty = true;
    for (uint64_t w : D[x]) empty = empty && !w;
    if (empty) {  // P_x is already I_x
      pl.state[x] = 2;
      continue;
    }
    if (express(D[x], zset)) final_row(x, true);
  }
  // nothing beyond peeling is determined (e.g. the unrecovered symbols lie in no received
  // equation's span): keep the peeling-only plan, no partial rows, no workspace
  bool gained = false;
  for (uint32_t m = 0; m < K && !gained; ++m) gained = pl.state[m] == 2;
  if (!gained) {
    for (uint32_t m = 0; m < K; ++m)
      if (!pl.state[m]) pl.level_of[m] = -1;
    pl.eliminated = 0;
    pl.inactivated = static_cast<uint32_t>(inact.size());
    pl.work_rows = 0;
    return FS_OK;
  }
  // emit the rows level by level after the DPG levels (stable within a level)
  int32_t any_recv = -1;
  for (uint32_t j = 0; j < n && any_recv < 0; ++j)
    if (received[j]) any_recv = static_cast<int32_t>(j);
  const size_t rows_before = pl.target.size();
  for (int32_t L = L0; L <= Lf; ++L) {
    for (const Row &r : rows) {
      if (r.level != L) continue;
      pl.target.push_back(r.target);
      pl.src.insert(pl.src.end(), r.src.begin(), r.src.end());
      if (r.src.empty()) {  // identically zero: XOR one received row with itself
        pl.src.push_back(static_cast<uint32_t>(any_recv) | kSrcCoded);
        pl.src.push_back(static_cast<uint32_t>(any_recv) | kSrcCoded);
      }
      pl.src.back() |= kSrcLast;
      pl.src_ptr.push_back(static_cast<int32_t>(pl.src.size()));
    }
    pl.level_ptr.push_back(static_cast<uint32_t>(pl.target.size()));
  }
  auto nonzero = [](const std::vector<uint64_t> &v) {
    for (uint64_t w : v)
      if (w) return true;
    return false;
  };
  for (uint32_t m = 0; m < K; ++m) {
    if (pl.state[m] == 2 && (kind[m] == 2 || nonzero(D[m]))) pl.level_of[m] = Lf;
    else if (!pl.state[m]) pl.level_of[m] = -1;
  }
  pl.eliminated = 0;
  for (uint32_t m = 0; m < K; ++m) pl.eliminated += pl.state[m] == 2 ? 1 : 0;
  pl.inactivated = ni;
  pl.work_rows = nz;
  (void)rows_before;
  return FS_OK;
}

}  // namespace

fs_status build_decode_plan(const Graph &g, const uint8_t *received, DecodePlan &pl, bool eliminate) {
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
  if (eliminate) return inactivation_phase(g, received, pl, members_fn(g), chosen_eq);
  return FS_OK;
}

}  // namespace fsb
