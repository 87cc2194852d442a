// Host-side seeded graph generator (step a1) and SMEM-kernel work scheduler.
//
// Graph (§2.2 steps (1) and (2); PAPER.md:95 seeded regeneration;
// PAPER.md:103 "c_d data node neighbors are selected"): one splitmix64 stream (reading R2)
// emits first the p precode checks (d_p distinct data indices each, R11) and then the n LT
// rows (one degree draw from Omega / RSD, then that many distinct indices in [0,K), R12),
// reading R5.  Indices: x mod range with rejection of duplicates (R6).  Degree: inverse
// CDF of u = (x >> 11) * 2^-53 over a CDF built in ascending order (R7-R10).  Rows are
// stored sorted (R14).  This file shares no code with oracle/ (DESIGN.md §2).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <queue>
#include <cstdlib>
#include <string>
#include <thread>

#include "fsb_internal.h"

namespace fsb {
namespace {

struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
};

// Distinct-index sampler with an epoch-stamped membership table (O(1) duplicate test).
struct NeighbourSampler {
  std::vector<uint32_t> stamp;
  uint32_t epoch = 0;
  explicit NeighbourSampler(uint32_t range) : stamp(range, 0) {}
  void draw(SplitMix64 &rng, uint32_t d, uint32_t range, int32_t *out) {
    if (++epoch == 0) {  // wrapped: clear
      std::fill(stamp.begin(), stamp.end(), 0);
      epoch = 1;
    }
    uint32_t got = 0;
    while (got < d) {
      uint32_t idx = static_cast<uint32_t>(rng.next() % static_cast<uint64_t>(range));
      if (stamp[idx] == epoch) continue;  // duplicate: redraw (R6)
      stamp[idx] = epoch;
      out[got++] = static_cast<int32_t>(idx);
    }
    std::sort(out, out + d);
  }
};

}  // namespace

// Largest prime factor by trial division (Alg 2's largest_prime_factor).
uint32_t lpf(uint32_t x) {
  uint32_t best = 1;
  for (uint32_t d = 2; static_cast<uint64_t>(d) * d <= x; ++d)
    while (x % d == 0) {
      best = d;
      x /= d;
    }
  return x > 1 ? x : best;
}

// Array LDPC shape for the paper's (b, k) = (k, K): {P, k', j'}; false if not realizable.
bool array_shape(uint32_t k, uint32_t K, uint32_t &P, uint32_t &kp, uint32_t &jp) {
  if (k == 0 || K <= k) return false;
  P = lpf(K);
  if (P < 2 || k % P) return false;
  kp = K / P;
  jp = kp - k / P;
  return jp >= 1 && kp > jp && kp <= P;
}

fs_status validate_params(const fs_params &prm) {
  if (prm.k == 0 || prm.n == 0) { set_error("k and n must be >= 1"); return FS_EINVAL; }
  if (prm.precode != FS_PRECODE_RANDOM && prm.precode != FS_PRECODE_ARRAY) {
    set_error("unknown precode kind");
    return FS_EINVAL;
  }
  if (prm.precode == FS_PRECODE_ARRAY) {
    uint32_t P, kp, jp;
    if (prm.p == 0 || static_cast<uint64_t>(prm.k) + prm.p >= (1ull << 31) ||
        !array_shape(prm.k, prm.k + prm.p, P, kp, jp)) {
      set_error("array precode not realizable: need P = largest prime factor of k+p dividing k, "
                "j' = (k+p)/P - k/P >= 1 and k/P >= 1, (k+p)/P <= P");
      return FS_EINVAL;
    }
  }
  if (prm.t == 0 || prm.t % 16 != 0) { set_error("t must be a positive multiple of 16"); return FS_EINVAL; }
  if (prm.t >= (1ull << 31)) { set_error("t must be below 2^31"); return FS_EINVAL; }
  if (prm.precode == FS_PRECODE_RANDOM && prm.p > 0 && (prm.d_p == 0 || prm.d_p > prm.k)) {
    set_error("precode degree d_p must satisfy 1 <= d_p <= k");
    return FS_EINVAL;
  }
  if (static_cast<uint64_t>(prm.k) + prm.p >= (1ull << 31)) { set_error("k+p too large"); return FS_EINVAL; }
  if (prm.files > 1 && prm.n % prm.files != 0) {
    set_error("per-file streams need files | n (PAPER.md:88)");
    return FS_EINVAL;
  }
  if (prm.dist != FS_DIST_RSD && prm.dist != FS_DIST_FINITE) { set_error("unknown distribution"); return FS_EDIST; }
  return FS_OK;
}

// CDF over the support, ascending (readings R7-R10, R15).  Returns FS_EDIST on bad input.
fs_status build_cdf(const fs_params &prm, std::vector<uint32_t> &deg, std::vector<double> &cdf) {
  const uint32_t K = prm.k + prm.p;
  std::vector<double> w;
  deg.clear();
  cdf.clear();
  if (prm.dist == FS_DIST_RSD) {
    // Robust Soliton (Luby) over K = k+p intermediate symbols (R10).
    const double c = prm.rsd_c, delta = prm.rsd_delta;
    if (!(c > 0.0)) { set_error("RSD c must be > 0"); return FS_EDIST; }
    if (!(delta > 0.0 && delta < 1.0)) { set_error("RSD delta must be in (0,1)"); return FS_EDIST; }
    const double R = c * std::log(static_cast<double>(K) / delta) * std::sqrt(static_cast<double>(K));
    if (!(R / delta > 1.0)) { set_error("RSD R/delta must exceed 1"); return FS_EDIST; }
    const double spike = std::floor(static_cast<double>(K) / R);
    if (spike < 1.0) { set_error("RSD spike K/R < 1"); return FS_EDIST; }
    const uint32_t m = static_cast<uint32_t>(spike);
    deg.resize(K);
    w.resize(K);
    for (uint32_t i = 1; i <= K; ++i) {
      const double rho = (i == 1) ? 1.0 / static_cast<double>(K)
                                  : 1.0 / (static_cast<double>(i) * static_cast<double>(i - 1));
      double tau = 0.0;
      if (i < m) tau = R / (static_cast<double>(i) * static_cast<double>(K));
      else if (i == m) tau = R * std::log(R / delta) / static_cast<double>(K);
      deg[i - 1] = i;
      w[i - 1] = rho + tau;
    }
  } else {
    // Finite max-degree Omega(x); degrees > K merged into K (R15).
    if (prm.fin_len == 0 || !prm.fin_deg || !prm.fin_prob) { set_error("empty distribution"); return FS_EDIST; }
    double sum = 0.0;
    for (uint32_t i = 0; i < prm.fin_len; ++i) {
      const uint32_t d = prm.fin_deg[i];
      const double q = prm.fin_prob[i];
      if (d == 0) { set_error("degree 0 in distribution"); return FS_EDIST; }
      if (i > 0 && d <= prm.fin_deg[i - 1]) { set_error("degrees must be strictly increasing"); return FS_EDIST; }
      if (!(q >= 0.0)) { set_error("negative probability"); return FS_EDIST; }
      sum += q;
      const uint32_t dc = std::min(d, K);
      if (!deg.empty() && deg.back() == dc) {
        w.back() += q;
      } else {
        deg.push_back(dc);
        w.push_back(q);
      }
    }
    if (std::fabs(sum - 1.0) > 1e-5) { set_error("probabilities must sum to 1 (within 1e-5)"); return FS_EDIST; }
  }
  double total = 0.0;
  for (double x : w) total += x;  // ascending degree order (R7)
  if (!(total > 0.0)) { set_error("distribution has zero mass"); return FS_EDIST; }
  cdf.resize(w.size());
  double acc = 0.0;
  for (size_t i = 0; i < w.size(); ++i) {
    acc = acc + w[i] / total;
    cdf[i] = acc;
  }
  cdf.back() = 1.0;
  return FS_OK;
}

fs_status generate_csr(Graph &g) {
  const fs_params &prm = g.prm;
  std::vector<uint32_t> deg;
  std::vector<double> cdf;
  fs_status st = build_cdf(prm, deg, cdf);
  if (st != FS_OK) return st;
  const uint32_t k = prm.k, p = prm.p, n = prm.n, K = k + p;
  SplitMix64 rng(prm.seed);
  NeighbourSampler sampler(K);
  // step (1): precode checks first (R5, R11); the array precode (Alg 2) draws nothing
  g.pre_row_ptr.assign(p + 1, 0);
  if (prm.precode == FS_PRECODE_ARRAY) {
    uint32_t P = 0, kp = 0, jp = 0;
    array_shape(k, K, P, kp, jp);
    const uint32_t d = kp - jp;
    g.prm.d_p = d;
    g.pre_col.assign(static_cast<size_t>(p) * d, 0);
    // Alg 2: check i + jP, member slot m-1; mod = non-negative residue (R18).
    // Member values index the K symbols: data m < k, check m-k (always an earlier check).
    uint32_t r = 0;
    for (uint32_t j = 0; j < jp; ++j)
      for (uint32_t i = 0; i < P; ++i, ++r) {
        for (uint32_t m = 1; m <= d; ++m) {
          const int64_t x = static_cast<int64_t>(m) * (static_cast<int64_t>(jp) - j - 1) - i - 1 + P;
          const int64_t res = ((x % P) + P) % P;
          g.pre_col[static_cast<size_t>(r) * d + m - 1] = static_cast<int32_t>(
              static_cast<int64_t>(kp) * P - (static_cast<int64_t>(jp) - j + m - 1) * P - res - 1);
        }
        g.pre_row_ptr[r + 1] = static_cast<int32_t>((r + 1) * d);
      }
  } else {
    g.pre_col.assign(static_cast<size_t>(p) * prm.d_p, 0);
    for (uint32_t i = 0; i < p; ++i) {
      sampler.draw(rng, prm.d_p, k, g.pre_col.data() + static_cast<size_t>(i) * prm.d_p);
      g.pre_row_ptr[i + 1] = static_cast<int32_t>((i + 1) * prm.d_p);
    }
  }
  // step (2): LT rows, one degree draw then the neighbour draws (R5, R12).  With s = files > 1
  // output file i (rows [i n/s, (i+1) n/s)) draws from its own stream seeded seed + i
  // (reading R17); file 0 continues the base stream after the precode draws, so
  // s = 1 is the single stream.  Files are independent: generated on parallel host threads.
  const uint32_t s = std::max<uint32_t>(prm.files, 1), rows_per = n / s;
  struct FileRows {
    std::vector<int32_t> col, len;
    uint32_t max_degree = 0;
  };
  std::vector<FileRows> files(s);
  auto gen_file = [&](uint32_t f, SplitMix64 frng, NeighbourSampler &smp) {
    FileRows &fr = files[f];
    fr.len.resize(rows_per);
    fr.col.reserve(static_cast<size_t>(rows_per) * 8);
    std::vector<int32_t> row;
    for (uint32_t j = 0; j < rows_per; ++j) {
      const uint64_t x = frng.next();
      const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
      const size_t idx = static_cast<size_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      uint32_t d = deg[std::min(idx, deg.size() - 1)];
      if (d > K) d = K;
      row.resize(d);
      smp.draw(frng, d, K, row.data());
      fr.col.insert(fr.col.end(), row.begin(), row.end());
      fr.len[j] = static_cast<int32_t>(d);
      fr.max_degree = std::max(fr.max_degree, d);
    }
  };
  if (s == 1) {
    gen_file(0, rng, sampler);
  } else {
    const uint32_t hw = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
    const uint32_t nthreads = std::min(s, hw);
    std::vector<std::thread> pool;
    for (uint32_t w = 0; w < nthreads; ++w)
      pool.emplace_back([&, w] {
        NeighbourSampler smp(K);
        for (uint32_t f = w; f < s; f += nthreads) gen_file(f, f == 0 ? rng : SplitMix64(prm.seed + f), smp);
      });
    for (auto &th : pool) th.join();
  }
  g.lt_row_ptr.assign(n + 1, 0);
  g.lt_col.clear();
  g.max_degree = 0;
  size_t nnz = 0;
  for (const FileRows &fr : files) nnz += fr.col.size();
  if (nnz >= (1ull << 31)) { set_error("graph too large (nnz >= 2^31)"); return FS_EINVAL; }
  g.lt_col.reserve(nnz);
  uint32_t j = 0;
  for (const FileRows &fr : files) {
    g.lt_col.insert(g.lt_col.end(), fr.col.begin(), fr.col.end());
    for (int32_t d : fr.len) {
      g.lt_row_ptr[j + 1] = g.lt_row_ptr[j] + d;
      ++j;
    }
    g.max_degree = std::max(g.max_degree, fr.max_degree);
  }
  return FS_OK;
}

fs_status validate_csr(const Graph &g) {
  const uint32_t k = g.prm.k, p = g.prm.p, n = g.prm.n, K = k + p;
  if (g.pre_row_ptr.size() != p + 1 || g.lt_row_ptr.size() != n + 1) { set_error("CSR row_ptr size"); return FS_EINVAL; }
  std::vector<uint32_t> seen(K, 0);
  uint32_t epoch = 0;
  // precode row r: members are data (< k) or earlier checks (k + r' with r' < r)
  auto check_rows = [&](const std::vector<int32_t> &rp, const std::vector<int32_t> &col, uint32_t rows,
                        bool precode) -> bool {
    if (rp[0] != 0) return false;
    for (uint32_t r = 0; r < rows; ++r) {
      if (rp[r + 1] < rp[r] || static_cast<size_t>(rp[r + 1]) > col.size()) return false;
      if (rp[r + 1] == rp[r]) return false;  // every row has degree >= 1
      // every precode row has exactly d_p members whatever the precode kind: the kernels index
      // member e of check c as pre_col[c*d_p + e] and size the staged member rows by p*d_p
      if (precode && static_cast<uint32_t>(rp[r + 1] - rp[r]) != g.prm.d_p) return false;
      ++epoch;
      for (int32_t e = rp[r]; e < rp[r + 1]; ++e) {
        const int32_t m = col[e];
        const uint32_t range = precode ? k + r : K;
        if (m < 0 || static_cast<uint32_t>(m) >= range) return false;
        if (seen[m] == epoch) return false;
        seen[m] = epoch;
      }
    }
    return static_cast<size_t>(rp[rows]) == col.size();
  };
  if (p && g.prm.precode == FS_PRECODE_ARRAY) {  // Alg 2's shape fixes the member count k'-j'
    uint32_t P = 0, kp = 0, jp = 0;
    if (!array_shape(k, K, P, kp, jp) || g.prm.d_p != kp - jp) {
      set_error("array precode CSR: members per check must be k'-j' of Alg 2");
      return FS_EINVAL;
    }
  }
  if (!check_rows(g.pre_row_ptr, g.pre_col, p, true)) { set_error("invalid precode CSR"); return FS_EINVAL; }
  if (!check_rows(g.lt_row_ptr, g.lt_col, n, false)) { set_error("invalid LT CSR"); return FS_EINVAL; }
  return FS_OK;
}

// Precode levels: a check reading only data is level 0, else 1 + the largest level of the
// checks it reads.  The kernels compute one level at a time, so levels must not decrease with
// the row index (true for the random precode, one level, and for Alg 2, level = block row j).
fs_status build_precode_levels(Graph &g) {
  const uint32_t k = g.prm.k, p = g.prm.p;
  std::vector<uint32_t> level(p, 0);
  g.pre_level_ptr.assign(1, 0);
  uint32_t cur = 0;
  for (uint32_t r = 0; r < p; ++r) {
    uint32_t L = 0;
    for (int32_t e = g.pre_row_ptr[r]; e < g.pre_row_ptr[r + 1]; ++e) {
      const uint32_t m = static_cast<uint32_t>(g.pre_col[e]);
      if (m >= k) L = std::max(L, level[m - k] + 1);
    }
    level[r] = L;
    if (r > 0 && L < cur) { set_error("precode levels must not decrease with the row index"); return FS_EINVAL; }
    while (cur < L) {
      g.pre_level_ptr.push_back(r);
      ++cur;
    }
  }
  g.pre_level_ptr.push_back(p);
  return FS_OK;
}

// ------------------------------------------------------------ SMEM kernel work schedule
// Degree-aware, edge-balanced, bank-conflict-free split of one tile's LT work over
// kConsumerWarps warps (record format and bank rule: fsb_internal.h).
//
// - Rows of degree in (kSplitThreshold, kSplit2Max] become pair-splits (evens in half 0, odds in
//   half 1 of one pair of groups); heavier rows become warp-split items: their even tile rows are
//   dealt round-robin to the 8 half-0 groups and their odd rows to the 8 half-1 groups.
// - Lighter rows are paired (A for half 0, B for half 1 of one pair): within a degree class,
//   rows are sorted by their number of even sources and the most-even row is paired with the
//   least-even one, so that A's evens meet B's odds and A's odds meet B's evens; leftovers are
//   matched with the zero row of the opposite parity.  Pairs are sorted by length and packed
//   8 per item (the item length is the longest pair's; shorter pairs pad with zero rows).
// - Items are dealt longest-first to the least loaded warp (LPT), an item costing its length
//   plus a per-item overhead (default 12 steps: same-box A/B of the 16-group items, config 4
//   0.5826 -> 0.5741 ms against 6, 20 ties; profiles/r02_s4/ab_groups16.txt).
void build_smem_schedule(Graph &g) {
  SmemSchedule &s = g.sched;
  s = SmemSchedule();
  g.smem_eligible = false;
  // warps for the precode (FSB_PRECODE_WARPS = 3..7 overrides): 3, or 5 when the precode is >= 5%
  // of the tile's gathers (array precode).  Same-box A/B (profiles/r02/ab_r02aj_precode_warps.txt):
  // config 6 (13.5%) 0.758 -> 0.717 ms with 5; configs 4 and 7 (0.4%) fastest with 3.
  {
    static const int pw_env = [] {
      const char *e = std::getenv("FSB_PRECODE_WARPS");
      return e ? std::atoi(e) : 0;
    }();
    int pw = g.pre_col.size() * 20 >= g.lt_col.size() ? 5 : kPrecodeWarps;
    if (pw_env >= 3 && pw_env <= 7) pw = pw_env;
    s.nconsumer = static_cast<uint32_t>(kConsumerWarps + kPrecodeWarps - pw);
  }
  const uint32_t k = g.prm.k, p = g.prm.p, n = g.prm.n;
  s.kpad = (k + kUnitRows - 1) / kUnitRows * kUnitRows;
  s.zero_even = (s.kpad + p + 1) & ~1u;
  s.tile_rows = s.zero_even + 2;
  s.data_units = s.kpad / kUnitRows;
  s.tile_units = (s.tile_rows + kUnitRows - 1) / kUnitRows;
  if (g.prm.t % kSliceBytes != 0 || g.prm.t > 0xFFFFFFFFull || n > kMaxSmemRows || s.tile_rows > kMaxSmemSlots) return;
  const uint16_t z0 = static_cast<uint16_t>(s.zero_even), z1 = static_cast<uint16_t>(s.zero_even + 1);
  auto slot = [&](int32_t m) -> uint16_t {
    const uint32_t r = static_cast<uint32_t>(m) < k ? static_cast<uint32_t>(m) : s.kpad + (m - k);
    return static_cast<uint16_t>(r);
  };
  s.pre_slots.resize(g.pre_col.size());
  for (size_t e = 0; e < g.pre_col.size(); ++e) s.pre_slots[e] = slot(g.pre_col[e]);  // data or earlier check

  struct Pair {                      // one group: half 0 (A) and half 1 (B)
    uint16_t row[2] = {kNoRow, kNoRow};
    std::vector<uint16_t> seq[2];    // seq[0][e] even <=> seq[1][e] odd
    bool split = false;              // pair-split: A and B hold the two parts of row[0]
  };
  constexpr int kPairsPerItem = kGroupsPerWarp / 2;
  struct Item {
    bool split = false;
    uint32_t len = 0;
    Pair grp[kPairsPerItem];
  };
  auto row_slots = [&](uint32_t j, std::vector<uint16_t> &ev, std::vector<uint16_t> &od) {
    for (int32_t e = g.lt_row_ptr[j]; e < g.lt_row_ptr[j + 1]; ++e) {
      const uint16_t v = slot(g.lt_col[e]);
      ((v & 1) ? od : ev).push_back(v);
    }
  };
  // pair rows A (half 0) and B (half 1; kNoRow = none) with parity-complementary steps
  auto make_pair = [&](uint32_t a, uint32_t b) {
    Pair pr;
    std::vector<uint16_t> ea, oa, eb, ob;
    row_slots(a, ea, oa);
    pr.row[0] = static_cast<uint16_t>(a);
    if (b != UINT32_MAX) {
      row_slots(b, eb, ob);
      pr.row[1] = static_cast<uint16_t>(b);
    }
    auto step = [&](uint16_t x, uint16_t y) {
      pr.seq[0].push_back(x);
      pr.seq[1].push_back(y);
    };
    size_t i = 0, j = 0;
    for (; i < ea.size() && j < ob.size(); ++i, ++j) step(ea[i], ob[j]);
    for (; i < ea.size(); ++i) step(ea[i], z1);
    size_t u = 0, v = 0;
    for (; u < oa.size() && v < eb.size(); ++u, ++v) step(oa[u], eb[v]);
    for (; u < oa.size(); ++u) step(oa[u], z0);
    for (; j < ob.size(); ++j) step(z0, ob[j]);
    for (; v < eb.size(); ++v) step(z1, eb[v]);
    return pr;
  };

  // split thresholds (FSB_SPLIT1 / FSB_SPLIT2 override kSplitThreshold / kSplit2Max: tuning)
  static const uint32_t split1 = [] {
    const char *e = std::getenv("FSB_SPLIT1");
    return e ? static_cast<uint32_t>(std::atoi(e)) : static_cast<uint32_t>(kSplitThreshold);
  }();
  static const uint32_t split2 = [] {
    const char *e = std::getenv("FSB_SPLIT2");
    return e ? static_cast<uint32_t>(std::atoi(e)) : static_cast<uint32_t>(kSplit2Max);
  }();
  std::vector<Item> items;
  std::vector<uint32_t> light;
  std::vector<Pair> pairs;
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t d = static_cast<uint32_t>(g.lt_row_ptr[j + 1] - g.lt_row_ptr[j]);
    if (d > split1 && d <= split2) {
      // pair-split: evens in half 0, odds in half 1 of one group
      Pair pr;
      pr.split = true;
      pr.row[0] = static_cast<uint16_t>(j);
      pr.row[1] = kNoRow;
      std::vector<uint16_t> ev, od;
      row_slots(j, ev, od);
      const size_t L = std::max(ev.size(), od.size());
      pr.seq[0] = ev;
      pr.seq[1] = od;
      pr.seq[0].resize(L, z0);
      pr.seq[1].resize(L, z1);
      pairs.push_back(std::move(pr));
      continue;
    }
    if (d > split1) {
      Item it;
      it.split = true;
      std::vector<uint16_t> ev, od;
      row_slots(j, ev, od);
      for (int q = 0; q < kPairsPerItem; ++q) {
        it.grp[q].row[0] = it.grp[q].row[1] = static_cast<uint16_t>(j);
        for (size_t e = q; e < ev.size(); e += kPairsPerItem) it.grp[q].seq[0].push_back(ev[e]);
        for (size_t e = q; e < od.size(); e += kPairsPerItem) it.grp[q].seq[1].push_back(od[e]);
      }
      for (int q = 0; q < kPairsPerItem; ++q) {
        it.len = std::max<uint32_t>(it.len, static_cast<uint32_t>(
                                                std::max(it.grp[q].seq[0].size(), it.grp[q].seq[1].size())));
      }
      for (int q = 0; q < kPairsPerItem; ++q) {
        it.grp[q].seq[0].resize(it.len, z0);
        it.grp[q].seq[1].resize(it.len, z1);
      }
      items.push_back(std::move(it));
    } else {
      light.push_back(j);
    }
  }
  // degree classes, each sorted by its rows' number of even sources; pair extremes
  auto degree = [&](uint32_t j) { return static_cast<uint32_t>(g.lt_row_ptr[j + 1] - g.lt_row_ptr[j]); };
  auto evens = [&](uint32_t j) {
    uint32_t c = 0;
    for (int32_t e = g.lt_row_ptr[j]; e < g.lt_row_ptr[j + 1]; ++e) c += (slot(g.lt_col[e]) & 1) ? 0 : 1;
    return c;
  };
  std::vector<uint32_t> ecount(n, 0);
  for (uint32_t j : light) ecount[j] = evens(j);
  std::stable_sort(light.begin(), light.end(), [&](uint32_t a, uint32_t b) {
    if (degree(a) != degree(b)) return degree(a) > degree(b);
    return ecount[a] < ecount[b];
  });
  // within a degree class d, a row with x even sources pairs best with one with d - x (its odds
  // then meet the partner's evens one for one): exact complements first, then the extremes of
  // what is left
  // The rows left after the exact complements of every class are matched across classes (greedy,
  // least parity padding; FSB_PAIR_GLOBAL=0: extremes within the class, the earlier rule).  Same
  // box (profiles/r02_s4c/ab_pair_global.txt): config 6 0.6838 -> 0.6757 ms, config 7 0.6313 ->
  // 0.6289, config 4 unchanged (its parity padding falls 498 -> 432 slots per tile, its length
  // padding rises 482 -> 548).
  static const int pair_global = [] {
    const char *e = std::getenv("FSB_PAIR_GLOBAL");
    return e ? std::atoi(e) : 1;
  }();
  std::vector<uint32_t> pool;
  uint32_t carry = UINT32_MAX;  // an unpaired row left over from the previous class
  for (size_t c0 = 0; c0 < light.size();) {
    size_t c1 = c0;
    while (c1 < light.size() && degree(light[c1]) == degree(light[c0])) ++c1;
    const uint32_t d = degree(light[c0]);
    std::vector<std::vector<uint32_t>> by_x(d + 1);
    for (size_t i = c0; i < c1; ++i) by_x[ecount[light[i]]].push_back(light[i]);
    for (uint32_t x = 0; 2 * x <= d; ++x) {
      std::vector<uint32_t> &a = by_x[x], &b = by_x[d - x];
      if (x == d - x) {
        while (a.size() >= 2) {
          const uint32_t r0 = a.back();
          a.pop_back();
          const uint32_t r1 = a.back();
          a.pop_back();
          pairs.push_back(make_pair(r0, r1));
        }
      } else {
        while (!a.empty() && !b.empty()) {
          pairs.push_back(make_pair(a.back(), b.back()));
          a.pop_back();
          b.pop_back();
        }
      }
    }
    std::vector<uint32_t> cls;
    if (carry != UINT32_MAX) cls.push_back(carry), carry = UINT32_MAX;
    for (uint32_t x = 0; x <= d; ++x) cls.insert(cls.end(), by_x[x].begin(), by_x[x].end());
    if (pair_global) {
      pool.insert(pool.end(), cls.begin(), cls.end());
      c0 = c1;
      continue;
    }
    std::stable_sort(cls.begin(), cls.end(), [&](uint32_t a, uint32_t b) { return ecount[a] < ecount[b]; });
    size_t lo = 0, hi = cls.size();
    while (hi - lo >= 2) {
      pairs.push_back(make_pair(cls[lo], cls[hi - 1]));
      ++lo;
      --hi;
    }
    if (hi - lo == 1) carry = cls[lo];
    c0 = c1;
  }
  if (carry != UINT32_MAX) pairs.push_back(make_pair(carry, UINT32_MAX));
  if (!pool.empty()) {
    // greedy: heaviest leftover first, its partner the unpaired leftover with the least parity
    // padding 2 (max(eA, oB) + max(oA, eB)) - dA - dB, ties to the closest degree; the scan looks
    // at the next kScan unpaired rows in degree order (a pool of n rows costs O(n kScan), not n^2)
    constexpr size_t kScan = 512;
    std::stable_sort(pool.begin(), pool.end(), [&](uint32_t a, uint32_t b) { return degree(a) > degree(b); });
    std::vector<char> used(pool.size(), 0);
    for (size_t i = 0; i < pool.size(); ++i) {
      if (used[i]) continue;
      used[i] = 1;
      const uint32_t a = pool[i], da = degree(a), ea = ecount[a], oa = da - ea;
      size_t best = SIZE_MAX;
      int64_t bcost = INT64_MAX;
      size_t seen = 0;
      for (size_t j = i + 1; j < pool.size() && seen < kScan; ++j) {
        if (used[j]) continue;
        ++seen;
        const uint32_t b = pool[j], db = degree(b), eb = ecount[b], ob = db - eb;
        const int64_t pad = 2 * static_cast<int64_t>(std::max(ea, ob) + std::max(oa, eb)) - da - db;
        const int64_t cost = pad * 4096 + (static_cast<int64_t>(da) - db);
        if (cost < bcost) bcost = cost, best = j;
      }
      if (best == SIZE_MAX) {
        pairs.push_back(make_pair(a, UINT32_MAX));
      } else {
        used[best] = 1;
        pairs.push_back(make_pair(a, pool[best]));
      }
    }
  }
  std::stable_sort(pairs.begin(), pairs.end(),
                   [](const Pair &a, const Pair &b) { return a.seq[0].size() > b.seq[0].size(); });
  for (size_t i = 0; i < pairs.size(); i += kPairsPerItem) {
    Item it;
    for (int q = 0; q < kPairsPerItem && i + q < pairs.size(); ++q) {
      it.grp[q] = pairs[i + q];
      it.len = std::max<uint32_t>(it.len, static_cast<uint32_t>(it.grp[q].seq[0].size()));
    }
    for (int q = 0; q < kPairsPerItem; ++q) {
      it.grp[q].seq[0].resize(it.len, z0);
      it.grp[q].seq[1].resize(it.len, z1);
    }
    items.push_back(std::move(it));
  }
  for (const Item &it : items)
    if (it.len > kMaxItemLen || it.len == 0) return;
  // LPT cost of an item in gather steps: L plus a per-item overhead (head load, dispatch, store);
  // FSB_ITEM_OVERHEAD overrides it (tuning experiments)
  static const uint32_t overhead = [] {
    const char *e = std::getenv("FSB_ITEM_OVERHEAD");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 12u;
  }();
  auto cost = [](const Item &it) { return it.len + overhead + (it.split ? 2u : 0u); };
  std::vector<uint32_t> order(items.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cost(items[a]) > cost(items[b]); });
  using Load = std::pair<uint64_t, int>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  const int ncw = static_cast<int>(s.nconsumer);
  for (int w = 0; w < ncw; ++w) heap.push({0, w});
  std::vector<std::vector<uint32_t>> per_warp(ncw);
  for (uint32_t idx : order) {
    Load l = heap.top();
    heap.pop();
    per_warp[l.second].push_back(idx);
    heap.push({l.first + cost(items[idx]), l.second});
  }
#ifdef FSB_EXPERIMENTS
  // profiling experiment (FSB_SCHED_DEBUG=zero): every slot reads a zero row of its half's parity
  // -- output is wrong by design, so it exists only in experiment builds (-DFSB_EXPERIMENTS)
  if (const char *dbg = std::getenv("FSB_SCHED_DEBUG")) {
    if (std::string(dbg) == "zero")
      for (Item &it : items)
        for (int q = 0; q < kPairsPerItem; ++q)
          for (int hh = 0; hh < 2; ++hh)
            for (uint16_t &v : it.grp[q].seq[hh]) v = hh ? z1 : z0;
  }
#endif
  // emit the two chunk streams, warp after warp (64 words per chunk; group g: words 4g..4g+3;
  // pair q, half hh in group 4(q>>1) + (q&1) + 2hh)
  s.warp_info.assign(ncw * 3, 0);
  std::vector<uint32_t> heads, conts;
  auto put = [](uint32_t &word, uint32_t i, uint16_t v) {  // slot i of a word pair position
    const uint32_t sh = (i & 1) ? kSlotHiShift : 0;
    word = (word & ~(((1u << kSlotBits) - 1) << sh)) | (static_cast<uint32_t>(v) << sh);
  };
  const uint32_t wpc = kChunkBytes / 4;  // words per chunk
  s.steps_max = s.steps_total = s.pad_slots = 0;
  for (int w = 0; w < ncw; ++w) {
    s.warp_info[w * 3 + 0] = static_cast<uint32_t>(per_warp[w].size());
    s.warp_info[w * 3 + 1] = static_cast<uint32_t>(heads.size() / wpc);
    s.warp_info[w * 3 + 2] = static_cast<uint32_t>(conts.size() / wpc);
    uint32_t steps = 0;
    for (uint32_t idx : per_warp[w]) {
      const Item &it = items[idx];
      bool item_pair_split = false;
      for (int q = 0; q < kPairsPerItem; ++q) item_pair_split = item_pair_split || it.grp[q].split;
      const size_t hb = heads.size();
      heads.resize(hb + wpc, 0);
      const uint32_t ncont = it.len > kHeadSlots ? (it.len - kHeadSlots + kChunkSlots - 1) / kChunkSlots : 0;
      const size_t cb = conts.size();
      conts.resize(cb + static_cast<size_t>(ncont) * wpc, 0);
      for (int h = 0; h < kGroupsPerWarp; ++h) {
        const int q = ((h >> 2) << 1) | (h & 1), hh = (h >> 1) & 1;  // pair, half
        const Pair &pr = it.grp[q];
        const std::vector<uint16_t> &seq = pr.seq[hh];
        heads[hb + h * 4] = static_cast<uint32_t>(pr.row[hh]) |
                            (static_cast<uint32_t>(it.len | (it.split ? kSplitBit : 0) |
                                                   (item_pair_split ? kPairSplitBit : 0))
                             << 16);
        if (pr.split) heads[hb + h * 4 + 1] |= kPairFlag;
        for (uint32_t e = 0; e < it.len; ++e) {
          if (seq[e] == z0 || seq[e] == z1) ++s.pad_slots;
          if (e < kHeadSlots) {
            put(heads[hb + h * 4 + 1 + e / 2], e, seq[e]);
          } else {
            const uint32_t f = e - kHeadSlots;
            put(conts[cb + (f / kChunkSlots) * wpc + h * 4 + (f % kChunkSlots) / 2], f, seq[e]);
          }
        }
        // unused slot positions of the last chunk: parity-correct zero rows (never read)
        const uint16_t zp = hh ? z1 : z0;
        for (uint32_t e = it.len; e < kHeadSlots + ncont * kChunkSlots; ++e) {
          if (e < kHeadSlots) {
            put(heads[hb + h * 4 + 1 + e / 2], e, zp);
          } else {
            const uint32_t f = e - kHeadSlots;
            put(conts[cb + (f / kChunkSlots) * wpc + h * 4 + (f % kChunkSlots) / 2], f, zp);
          }
        }
      }
      steps += it.len;
    }
    s.steps_max = std::max(s.steps_max, steps);
    s.steps_total += steps;
  }
  heads.resize(heads.size() + kStreamPad * wpc, 0);
  conts.resize(conts.size() + kStreamPad * wpc, 0);
  s.cont_base = static_cast<uint32_t>(heads.size() / wpc);
  s.words = std::move(heads);
  s.words.insert(s.words.end(), conts.begin(), conts.end());
  g.smem_eligible = true;
}

// Pack the LT rows into the fixed-size edge windows of fsb_lt_win (fsb_internal.h: LtWindows):
// rows in order, a window closes when the next row would exceed 32 x regs edges (after padding
// to a multiple of 4) or max_rows rows.  A row of more than 32 x regs - 3 edges fits no window:
// then count = 0 and the band kernels take every call.
void build_lt_windows(Graph &g, uint32_t max_rows, uint32_t regs) {
  LtWindows &w = g.win;
  w = LtWindows();
  const uint32_t kWinEntries = 32 * regs;
  w.entries = kWinEntries;
  const uint32_t n = g.prm.n;
  const std::vector<int32_t> &rp = g.lt_row_ptr;
  if (max_rows == 0) return;
  for (uint32_t j = 0; j < n; ++j)
    if (static_cast<uint32_t>(rp[j + 1] - rp[j]) + 3 > kWinEntries) return;
  uint32_t j = 0;
  while (j < n) {
    uint32_t j1 = j, cnt = 0;
    while (j1 < n && j1 - j < max_rows) {
      const uint32_t d = static_cast<uint32_t>(rp[j1 + 1] - rp[j1]);
      if (((cnt + d + 3) & ~3u) > kWinEntries) break;
      cnt += d;
      ++j1;
    }
    const uint32_t padded = (cnt + 3) & ~3u, skip = padded - cnt;
    const size_t base = w.ent.size();
    w.ent.resize(base + kWinEntries, 0u);
    for (uint32_t e = 0; e < skip; ++e) w.ent[base + e] = kWinSkip;
    uint32_t e = skip;
    for (uint32_t r = j; r < j1; ++r) {
      for (int32_t x = rp[r]; x < rp[r + 1]; ++x) w.ent[base + e++] = static_cast<uint32_t>(g.lt_col[x]);
      w.ent[base + e - 1] |= 0x80000000u;  // last edge of row r
    }
    w.hdr.push_back(j);
    w.hdr.push_back(padded / 4);
    j = j1;
  }
  w.count = static_cast<uint32_t>(w.hdr.size() / 2);
}

}  // namespace fsb
