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

// Residual GF(2) elimination after peeling ("needs an inactivation / GF(2)
// fallback at these overheads"; not in the paper, whose decoder is BP only).  The residual system:
// every received LT row and every precode check that still has an unknown, over the unknown
// symbols, each row augmented with its own equation index.  Gauss-Jordan to reduced row echelon
// form; a row whose unknown part is a unit vector e_c determines c (exactly the symbols in the
// row space, as the oracle's elimination), as the XOR of the equations in its augmented part:
// c = XOR over those e of (Y_e if an LT row) and of every known member, mod 2.  These rows form one
// final level (their sources are received rows and symbols recovered by peeling).
fs_status eliminate_residual(const Graph &g, const uint8_t *received, DecodePlan &pl, const Members &members) {
  const uint32_t n = g.prm.n, p = g.prm.p, K = g.prm.k + p;
  std::vector<int32_t> col_of(K, -1);
  std::vector<uint32_t> unk;
  for (uint32_t m = 0; m < K; ++m)
    if (!pl.state[m]) col_of[m] = static_cast<int32_t>(unk.size()), unk.push_back(m);
  const uint32_t u = static_cast<uint32_t>(unk.size());
  if (!u) return FS_OK;
  std::vector<uint32_t> eqs;
  for (uint32_t e = 0; e < n + p; ++e) {
    if (e < n && !received[e]) continue;
    bool any = false;
    members(e, [&](uint32_t m) { any = any || !pl.state[m]; });
    if (any) eqs.push_back(e);
  }
  const uint32_t q = static_cast<uint32_t>(eqs.size());
  if (static_cast<uint64_t>(u) * q > (1ull << 28)) {  // ~32 MB of bits: leave the residual
    pl.elim_skipped = 1;
    return FS_OK;
  }
  const uint32_t W1 = (u + 63) / 64, W2 = (q + 63) / 64, W = W1 + W2;
  std::vector<uint64_t> M(static_cast<size_t>(q) * W, 0);
  for (uint32_t r = 0; r < q; ++r) {
    uint64_t *row = &M[static_cast<size_t>(r) * W];
    members(eqs[r], [&](uint32_t m) {
      if (!pl.state[m]) row[col_of[m] >> 6] ^= 1ull << (col_of[m] & 63);
    });
    row[W1 + (r >> 6)] |= 1ull << (r & 63);
  }
  uint32_t piv = 0;
  std::vector<int32_t> pivcol;
  for (uint32_t c = 0; c < u && piv < q; ++c) {
    const uint32_t w = c >> 6;
    const uint64_t bit = 1ull << (c & 63);
    uint32_t r = piv;
    while (r < q && !(M[static_cast<size_t>(r) * W + w] & bit)) ++r;
    if (r == q) continue;
    if (r != piv)
      std::swap_ranges(M.begin() + static_cast<size_t>(r) * W, M.begin() + static_cast<size_t>(r + 1) * W,
                       M.begin() + static_cast<size_t>(piv) * W);
    const uint64_t *pr = &M[static_cast<size_t>(piv) * W];
    for (uint32_t o = 0; o < q; ++o) {
      if (o == piv) continue;
      uint64_t *ro = &M[static_cast<size_t>(o) * W];
      if (ro[w] & bit)
        for (uint32_t x = w; x < W; ++x) ro[x] ^= pr[x];  // words below w are zero in the pivot row
    }
    pivcol.push_back(static_cast<int32_t>(c));
    ++piv;
  }
  // rows whose unknown part is exactly e_c
  std::vector<uint8_t> parity(K, 0);
  std::vector<uint32_t> touched;
  int32_t any_recv = -1;
  for (uint32_t j = 0; j < n && any_recv < 0; ++j)
    if (received[j]) any_recv = static_cast<int32_t>(j);
  const size_t rows_before = pl.target.size();
  for (uint32_t r = 0; r < piv; ++r) {
    const uint64_t *row = &M[static_cast<size_t>(r) * W];
    uint32_t pop = 0;
    for (uint32_t x = 0; x < W1 && pop < 2; ++x) pop += static_cast<uint32_t>(__builtin_popcountll(row[x]));
    if (pop != 1) continue;
    const uint32_t c = unk[pivcol[r]];
    pl.target.push_back(static_cast<int32_t>(c));
    const size_t s0 = pl.src.size();
    for (uint32_t x = 0; x < W2; ++x)
      for (uint64_t bits = row[W1 + x]; bits; bits &= bits - 1) {
        const uint32_t e = eqs[x * 64 + static_cast<uint32_t>(__builtin_ctzll(bits))];
        if (e < n) pl.src.push_back(e | kSrcCoded);
        members(e, [&](uint32_t m) {
          if (pl.state[m] == 1) {
            if (!parity[m]) touched.push_back(m);
            parity[m] ^= 1;
          }
        });
      }
    for (uint32_t m : touched) {
      if (parity[m]) pl.src.push_back(m);
      parity[m] = 0;
    }
    touched.clear();
    if (pl.src.size() == s0) {  // identically zero: XOR one received row with itself
      pl.src.push_back(static_cast<uint32_t>(any_recv) | kSrcCoded);
      pl.src.push_back(static_cast<uint32_t>(any_recv) | kSrcCoded);
    }
    pl.src.back() |= kSrcLast;
    pl.src_ptr.push_back(static_cast<int32_t>(pl.src.size()));
  }
  if (pl.target.size() > rows_before) {
    const int32_t L = static_cast<int32_t>(pl.level_ptr.size()) - 1;
    for (size_t r = rows_before; r < pl.target.size(); ++r) {
      pl.state[pl.target[r]] = 2;
      pl.level_of[pl.target[r]] = L;
    }
    pl.level_ptr.push_back(static_cast<uint32_t>(pl.target.size()));
    pl.eliminated = static_cast<uint32_t>(pl.target.size() - rows_before);
  }
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
  if (eliminate) return eliminate_residual(g, received, pl, members_fn(g));
  return FS_OK;
}

}  // namespace fsb
