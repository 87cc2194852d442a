// Repair, update and degraded read: host side.
//
// 1. CGA, Algorithm 4 on B in F2^{K x n} (column j = the neighbours of coded
//    symbol j; the paper's k is our K = k+p, reading R19), with L^{(2,3)} = I_n carried along.
//    Exact sequential semantics of the pseudocode (j outer, i inner, b_j updated in place) on
//    sparse columns: the update test w(b_j ^ b_i) < w(b_j) is 2|b_j & b_i| > w(b_i), so only
//    columns overlapping b_j can qualify; their overlap counts are kept current through a
//    symbol -> columns index while b_j changes, and the candidates (2 cnt > w) are scanned in
//    ascending i from a bitset.  Identical output to the dense oracle (tests/test_repair.py).
// 2. The local sets: weight-0 column j -> Group #3 {C_s : l_{s,j}}, weight-1
//    column (symbol x) -> Group #2 (x, {C_s}); the §2.5 derived Group #3 sets (PAPER.md:245-260,
//    FS_CHECKS_M1 / FS_CHECKS_M2, setXOR); serialised in the <filename>_check.data format
//    (PAPER.md:311-320), smallest cardinality first (ties: reading R20).
// 3. The repair plan (reading R21): rounds of [one sweep over the Group #3 sets:
//    a set with exactly one unknown member repairs it; one sweep over the unknown coded symbols
//    ascending: C_j = XOR over its neighbours x of XOR(G_x) when every x has a Group #2 set whose
//    members are all known], then the wanted intermediate symbols (degraded read)
//    from their first available G_x.  Rows are grouped in levels (1 + max level of the sources)
//    and run by the same per-level gather-XOR kernel as the decoder (fsb_dpg_level).
#include <algorithm>
#include <cstring>

#include "fsb_internal.h"

namespace fsb {

namespace {

// symmetric difference of two ascending lists into out (ascending)
void sym_diff(const std::vector<int32_t> &a, const std::vector<int32_t> &b, std::vector<int32_t> &out) {
  out.clear();
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    if (a[i] < b[j]) out.push_back(a[i++]);
    else if (b[j] < a[i]) out.push_back(b[j++]);
    else ++i, ++j;
  }
  out.insert(out.end(), a.begin() + i, a.end());
  out.insert(out.end(), b.begin() + j, b.end());
}

struct Bitset {
  std::vector<uint64_t> w;
  explicit Bitset(size_t n) : w((n + 63) / 64, 0) {}
  void set(size_t i) { w[i >> 6] |= 1ull << (i & 63); }
  void clear(size_t i) { w[i >> 6] &= ~(1ull << (i & 63)); }
  size_t next(size_t i, size_t n) const {  // first set bit >= i, or n
    if (i >= n) return n;
    size_t q = i >> 6;
    uint64_t m = w[q] & (~0ull << (i & 63));
    for (;;) {
      if (m) return std::min(n, (q << 6) + static_cast<size_t>(__builtin_ctzll(m)));
      if (++q >= w.size()) return n;
      m = w[q];
    }
  }
};

}  // namespace

fs_status run_cga(const Graph &g, CgaResult &r) {
  const uint32_t n = g.prm.n, K = g.prm.k + g.prm.p;
  r = CgaResult();
  std::vector<std::vector<int32_t>> &b = r.b, &l = r.l;
  b.resize(n);
  l.resize(n);
  std::vector<uint32_t> w(n);
  std::vector<std::vector<uint32_t>> inv(K);
  for (uint32_t j = 0; j < n; ++j) {
    b[j].assign(g.lt_col.begin() + g.lt_row_ptr[j], g.lt_col.begin() + g.lt_row_ptr[j + 1]);
    std::sort(b[j].begin(), b[j].end());
    w[j] = static_cast<uint32_t>(b[j].size());
    for (int32_t x : b[j]) inv[x].push_back(j);
    l[j].assign(1, static_cast<int32_t>(j));
  }
  uint64_t zero = 0;
  for (uint32_t j = 0; j < n; ++j) zero += w[j] == 0;
  std::vector<uint32_t> cnt(n, 0), touched;
  std::vector<uint32_t> inbj(K, UINT32_MAX);  // inbj[x] == j <=> x in b_j (current j)
  Bitset cand(n);
  std::vector<int32_t> scratch;
  auto refresh = [&](uint32_t c) {
    if (2 * cnt[c] > w[c]) cand.set(c);
    else cand.clear(c);
  };
  while (static_cast<int64_t>(zero) < static_cast<int64_t>(n) - static_cast<int64_t>(K)) {
    ++r.sweeps;
    bool temp = false;
    for (uint32_t j = 0; j < n; ++j) {
      if (w[j] == 0) continue;  // 2 w(b_j) > w(b_i) never holds
      touched.clear();
      for (int32_t x : b[j]) {
        inbj[x] = j;
        for (uint32_t c : inv[x])
          if (c != j && cnt[c]++ == 0) touched.push_back(c);
      }
      for (uint32_t c : touched) refresh(c);
      for (size_t i = cand.next(0, n); i < n; i = cand.next(i + 1, n)) {
        if (!(2 * w[j] > w[i])) continue;
        // b_j ^= b_i (overlap counts of the other columns follow each toggled symbol)
        for (int32_t x : b[i]) {
          const bool removing = inbj[x] == j;
          for (uint32_t c : inv[x]) {
            if (c == j) continue;
            if (removing) --cnt[c];
            else if (cnt[c]++ == 0) touched.push_back(c);
            refresh(c);
          }
          auto &lst = inv[x];
          if (removing) {
            lst.erase(std::find(lst.begin(), lst.end(), j));
            inbj[x] = UINT32_MAX;
          } else {
            lst.push_back(j);
            inbj[x] = j;
          }
        }
        sym_diff(b[j], b[i], scratch);
        b[j].swap(scratch);
        w[j] = static_cast<uint32_t>(b[j].size());
        sym_diff(l[j], l[i], scratch);
        l[j].swap(scratch);
        temp = true;
        ++r.updates;
        if (w[j] == 0) {
          ++zero;
          break;  // no further i can qualify
        }
      }
      for (uint32_t c : touched) {
        cnt[c] = 0;
        cand.clear(c);
      }
      for (int32_t x : b[j]) inbj[x] = UINT32_MAX;
    }
    if (!temp) break;
  }
  r.zero_columns = static_cast<uint32_t>(zero);
  for (uint32_t j = 0; j < n; ++j) r.weight1_columns += w[j] == 1;
  return FS_OK;
}

fs_status build_check_data(const Graph &g, uint32_t flags, ChecksData &cd) {
  const uint32_t n = g.prm.n, k = g.prm.k, p = g.prm.p;
  cd = ChecksData();
  CgaResult r;
  fs_status st = run_cga(g, r);
  if (st != FS_OK) return st;
  cd.sweeps = r.sweeps;
  cd.zero_columns = r.zero_columns;
  cd.weight1_columns = r.weight1_columns;
  struct Group {
    int32_t x;  // -1: Group #3
    uint64_t key;
    std::vector<int32_t> mem;
  };
  std::vector<Group> groups;
  for (uint32_t j = 0; j < n; ++j) {
    if (r.b[j].size() == 0) groups.push_back({-1, j, r.l[j]});
    else if (r.b[j].size() == 1) groups.push_back({r.b[j][0], j, r.l[j]});
  }
  auto order = [](const Group &a, const Group &b) {
    return a.mem.size() != b.mem.size() ? a.mem.size() < b.mem.size() : a.key < b.key;
  };
  // G_x: the first Group #2 set of each symbol in (cardinality, key) order (reading R20)
  std::vector<const std::vector<int32_t> *> gx(k + p, nullptr);
  {
    std::vector<const Group *> sorted;
    for (const Group &gr : groups) sorted.push_back(&gr);
    std::sort(sorted.begin(), sorted.end(), [&](const Group *a, const Group *b) { return order(*a, *b); });
    for (const Group *gr : sorted)
      if (gr->x >= 0 && !gx[gr->x]) gx[gr->x] = &gr->mem;
  }
  std::vector<std::vector<int32_t>> derived;
  std::vector<int32_t> acc, tmp;
  if (flags & FS_CHECKS_M1) {  // degree-one coded node j with neighbour x
    for (uint32_t j = 0; j < n; ++j) {
      if (g.lt_row_ptr[j + 1] - g.lt_row_ptr[j] != 1) continue;
      const int32_t x = g.lt_col[g.lt_row_ptr[j]];
      if (!gx[x]) continue;
      sym_diff(*gx[x], std::vector<int32_t>{static_cast<int32_t>(j)}, acc);
      if (!acc.empty()) derived.push_back(acc);
    }
  }
  if (flags & FS_CHECKS_M2) {  // check #1 group -> setXOR of the G_x (Eq 4)
    for (uint32_t i = 0; i < p; ++i) {
      std::vector<int32_t> grp(g.pre_col.begin() + g.pre_row_ptr[i], g.pre_col.begin() + g.pre_row_ptr[i + 1]);
      grp.push_back(static_cast<int32_t>(k + i));
      bool all = true;
      for (int32_t x : grp) all = all && gx[x] != nullptr;
      if (!all) continue;
      acc.clear();
      for (int32_t x : grp) {
        sym_diff(acc, *gx[x], tmp);
        acc.swap(tmp);
      }
      if (!acc.empty()) derived.push_back(acc);
    }
  }
  for (size_t m = 0; m < derived.size(); ++m) groups.push_back({-1, n + m, std::move(derived[m])});
  cd.derived = static_cast<uint32_t>(derived.size());
  std::stable_sort(groups.begin(), groups.end(), order);
  for (const Group &gr : groups) {
    if (gr.x < 0) {
      cd.data.push_back(0);
      ++cd.group3;
    } else {
      cd.data.push_back(1);
      cd.data.push_back(gr.x);
      ++cd.group2;
    }
    cd.data.push_back(static_cast<int32_t>(gr.mem.size()));
    cd.data.insert(cd.data.end(), gr.mem.begin(), gr.mem.end());
  }
  return FS_OK;
}

fs_status parse_check_data(const Graph &g, const int32_t *data, uint64_t len, ChecksData &cd) {
  const uint32_t n = g.prm.n, K = g.prm.k + g.prm.p;
  cd = ChecksData();
  cd.data.assign(data, data + len);
  uint64_t i = 0;
  while (i < len) {
    const int32_t flag = data[i];
    if (flag != 0 && flag != 1) { set_error("check data: flag must be 0 or 1"); return FS_EINVAL; }
    if (flag == 1) {
      if (i + 1 >= len || data[i + 1] < 0 || static_cast<uint32_t>(data[i + 1]) >= K) {
        set_error("check data: Group #2 symbol out of range");
        return FS_EINVAL;
      }
      ++i;
    }
    if (i + 1 >= len) { set_error("check data: truncated"); return FS_EINVAL; }
    const int32_t d = data[i + 1];
    if (d < 1 || i + 2 + static_cast<uint64_t>(d) > len) { set_error("check data: bad set size"); return FS_EINVAL; }
    for (int32_t m = 0; m < d; ++m) {
      const int32_t c = data[i + 2 + m];
      if (c < 0 || static_cast<uint32_t>(c) >= n) { set_error("check data: coded index out of range"); return FS_EINVAL; }
    }
    if (flag) ++cd.group2;
    else ++cd.group3;
    i += 2 + static_cast<uint64_t>(d);
  }
  return FS_OK;
}

fs_status build_repair_plan(const Graph &g, const ChecksData &cd, const uint8_t *erased, const uint32_t *want,
                            uint32_t nwant, DecodePlan &pl, RepairStats &rs) {
  const uint32_t n = g.prm.n, K = g.prm.k + g.prm.p;
  pl = DecodePlan();
  pl.k = g.prm.k, pl.p = g.prm.p, pl.n = n, pl.K = K, pl.t = g.prm.t;
  rs = RepairStats();
  // the local sets, in array order
  std::vector<uint64_t> s3_off;  // offsets of Group #3 member lists into cd.data
  std::vector<std::vector<uint64_t>> s2_of(K);  // Group #2 sets of symbol x, array order
  for (uint64_t i = 0; i < cd.data.size();) {
    if (cd.data[i] == 0) {
      s3_off.push_back(i + 1);
      i += 2 + static_cast<uint64_t>(cd.data[i + 1]);
    } else {
      const int32_t x = cd.data[i + 1];
      if (static_cast<uint32_t>(x) < K) s2_of[x].push_back(i + 2);
      i += 3 + static_cast<uint64_t>(cd.data[i + 2]);
    }
  }
  auto members = [&](uint64_t off) { return std::make_pair(&cd.data[off + 1], cd.data[off]); };
  std::vector<uint8_t> unknown(n, 0);
  std::vector<int32_t> level(n, 0);
  uint32_t nunknown = 0;
  for (uint32_t j = 0; j < n; ++j)
    if (erased[j]) unknown[j] = 1, ++nunknown;
  rs.erased = nunknown;
  struct Step {
    int32_t target;  // coded j, or x | kSrcCoded-free intermediate flagged below
    bool coded;
    std::vector<int32_t> src;
    int32_t level;
  };
  std::vector<Step> steps;
  auto level_of = [&](const std::vector<int32_t> &src) {
    int32_t L = 0;
    for (int32_t c : src) L = std::max(L, level[c]);
    return L + 1;
  };
  auto avail_g2 = [&](uint32_t x) -> int64_t {
    for (uint64_t off : s2_of[x]) {
      auto [m, d] = members(off);
      bool ok = true;
      for (int32_t e = 0; e < d && ok; ++e) ok = !unknown[m[e]];
      if (ok) return static_cast<int64_t>(off);
    }
    return -1;
  };
  std::vector<int32_t> acc, tmp, part;
  bool progress = true;
  while (progress && nunknown) {
    progress = false;
    for (uint64_t off : s3_off) {  // A: Group #3 sets with exactly one unknown member
      auto [m, d] = members(off);
      int32_t miss = -1, nmiss = 0;
      for (int32_t e = 0; e < d && nmiss < 2; ++e)
        if (unknown[m[e]]) miss = m[e], ++nmiss;
      if (nmiss != 1) continue;
      Step s{miss, true, {}, 0};
      for (int32_t e = 0; e < d; ++e)
        if (m[e] != miss) s.src.push_back(m[e]);
      s.level = level_of(s.src);
      level[miss] = s.level;
      unknown[miss] = 0;
      --nunknown;
      steps.push_back(std::move(s));
      progress = true;
    }
    std::vector<uint32_t> snapshot;
    for (uint32_t j = 0; j < n; ++j)
      if (unknown[j]) snapshot.push_back(j);
    for (uint32_t j : snapshot) {  // B: C_j = XOR of the G_x of its neighbours
      if (!unknown[j]) continue;
      acc.clear();
      bool ok = true;
      for (int32_t e = g.lt_row_ptr[j]; e < g.lt_row_ptr[j + 1] && ok; ++e) {
        const int64_t off = avail_g2(static_cast<uint32_t>(g.lt_col[e]));
        if (off < 0) { ok = false; break; }
        auto [m, d] = members(static_cast<uint64_t>(off));
        part.assign(m, m + d);
        std::sort(part.begin(), part.end());
        sym_diff(acc, part, tmp);
        acc.swap(tmp);
      }
      if (!ok) continue;
      Step s{static_cast<int32_t>(j), true, acc, 0};
      s.level = level_of(s.src);
      level[j] = s.level;
      unknown[j] = 0;
      --nunknown;
      steps.push_back(std::move(s));
      progress = true;
    }
  }
  rs.unrepaired = nunknown;
  rs.repaired = rs.erased - nunknown;
  for (uint32_t r = 0; r < nwant; ++r) {  // C: degraded read of intermediate symbols
    if (want[r] >= K) { set_error("wanted symbol out of range"); return FS_EINVAL; }
    const int64_t off = avail_g2(want[r]);
    if (off < 0) { ++rs.want_missing; continue; }
    auto [m, d] = members(static_cast<uint64_t>(off));
    Step s{static_cast<int32_t>(want[r]), false, std::vector<int32_t>(m, m + d), 0};
    s.level = level_of(s.src);
    steps.push_back(std::move(s));
  }
  // a source-free recipe is the all-zero symbol: XOR a known symbol twice
  int32_t any_known = -1;
  for (uint32_t j = 0; j < n && any_known < 0; ++j)
    if (!erased[j]) any_known = static_cast<int32_t>(j);
  // GPU rows: by level, step order within a level
  int32_t maxL = 0;
  for (const Step &s : steps) maxL = std::max(maxL, s.level);
  pl.level_ptr.assign(1, 0);
  pl.src_ptr.assign(1, 0);
  for (int32_t L = 1; L <= maxL; ++L) {
    for (const Step &s : steps) {
      if (s.level != L) continue;
      pl.target.push_back(s.coded ? static_cast<int32_t>(static_cast<uint32_t>(s.target) | kSrcCoded) : s.target);
      if (s.src.empty()) {
        if (any_known < 0) { set_error("no known coded symbol"); return FS_EINVAL; }
        pl.src.push_back(static_cast<uint32_t>(any_known) | kSrcCoded);
        pl.src.push_back(static_cast<uint32_t>(any_known) | kSrcCoded);
      }
      for (int32_t c : s.src) pl.src.push_back(static_cast<uint32_t>(c) | kSrcCoded);
      pl.src.back() |= kSrcLast;
      pl.src_ptr.push_back(static_cast<int32_t>(pl.src.size()));
      rs.xor_sources += s.src.size();
    }
    pl.level_ptr.push_back(static_cast<uint32_t>(pl.target.size()));
  }
  rs.levels = static_cast<uint32_t>(maxL);
  rs.rows = static_cast<uint32_t>(pl.target.size());
  return FS_OK;
}

}  // namespace fsb
