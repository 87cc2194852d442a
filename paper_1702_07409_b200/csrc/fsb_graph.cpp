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

fs_status validate_params(const fs_params &prm) {
  if (prm.k == 0 || prm.n == 0) { set_error("k and n must be >= 1"); return FS_EINVAL; }
  if (prm.t == 0 || prm.t % 16 != 0) { set_error("t must be a positive multiple of 16"); return FS_EINVAL; }
  if (prm.p > 0 && (prm.d_p == 0 || prm.d_p > prm.k)) {
    set_error("precode degree d_p must satisfy 1 <= d_p <= k");
    return FS_EINVAL;
  }
  if (static_cast<uint64_t>(prm.k) + prm.p >= (1ull << 31)) { set_error("k+p too large"); return FS_EINVAL; }
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
  // step (1): precode checks first (R5, R11)
  g.pre_row_ptr.assign(p + 1, 0);
  g.pre_col.assign(static_cast<size_t>(p) * prm.d_p, 0);
  for (uint32_t i = 0; i < p; ++i) {
    sampler.draw(rng, prm.d_p, k, g.pre_col.data() + static_cast<size_t>(i) * prm.d_p);
    g.pre_row_ptr[i + 1] = static_cast<int32_t>((i + 1) * prm.d_p);
  }
  // step (2): LT rows, one degree draw then the neighbour draws (R5, R12)
  g.lt_row_ptr.assign(n + 1, 0);
  g.lt_col.clear();
  g.lt_col.reserve(static_cast<size_t>(n) * 8);
  g.max_degree = 0;
  std::vector<int32_t> row;
  for (uint32_t j = 0; j < n; ++j) {
    const uint64_t x = rng.next();
    const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
    const size_t idx = static_cast<size_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    uint32_t d = deg[std::min(idx, deg.size() - 1)];
    if (d > K) d = K;
    row.resize(d);
    sampler.draw(rng, d, K, row.data());
    g.lt_col.insert(g.lt_col.end(), row.begin(), row.end());
    if (g.lt_col.size() >= (1ull << 31)) { set_error("graph too large (nnz >= 2^31)"); return FS_EINVAL; }
    g.lt_row_ptr[j + 1] = static_cast<int32_t>(g.lt_col.size());
    g.max_degree = std::max(g.max_degree, d);
  }
  return FS_OK;
}

fs_status validate_csr(const Graph &g) {
  const uint32_t k = g.prm.k, p = g.prm.p, n = g.prm.n, K = k + p;
  if (g.pre_row_ptr.size() != p + 1 || g.lt_row_ptr.size() != n + 1) { set_error("CSR row_ptr size"); return FS_EINVAL; }
  std::vector<uint32_t> seen(K, 0);
  uint32_t epoch = 0;
  auto check_rows = [&](const std::vector<int32_t> &rp, const std::vector<int32_t> &col, uint32_t rows,
                        uint32_t range, bool fixed_deg) -> bool {
    if (rp[0] != 0) return false;
    for (uint32_t r = 0; r < rows; ++r) {
      if (rp[r + 1] < rp[r] || static_cast<size_t>(rp[r + 1]) > col.size()) return false;
      if (rp[r + 1] == rp[r]) return false;  // every row has degree >= 1
      if (fixed_deg && static_cast<uint32_t>(rp[r + 1] - rp[r]) != g.prm.d_p) return false;
      ++epoch;
      for (int32_t e = rp[r]; e < rp[r + 1]; ++e) {
        const int32_t m = col[e];
        if (m < 0 || static_cast<uint32_t>(m) >= range) return false;
        if (seen[m] == epoch) return false;
        seen[m] = epoch;
      }
    }
    return static_cast<size_t>(rp[rows]) == col.size();
  };
  if (!check_rows(g.pre_row_ptr, g.pre_col, p, k, true)) { set_error("invalid precode CSR"); return FS_EINVAL; }
  if (!check_rows(g.lt_row_ptr, g.lt_col, n, K, false)) { set_error("invalid LT CSR"); return FS_EINVAL; }
  return FS_OK;
}

// ------------------------------------------------------------ SMEM kernel work schedule
// Degree-aware, edge-balanced split of one tile's LT work over kConsumerWarps warps (format:
// SmemSchedule in fsb_internal.h).
void build_smem_schedule(Graph &g) {
  SmemSchedule &s = g.sched;
  s = SmemSchedule();
  g.smem_eligible = false;
  const uint32_t k = g.prm.k, p = g.prm.p, n = g.prm.n;
  s.kpad = (k + kUnitRows - 1) / kUnitRows * kUnitRows;
  s.data_units = s.kpad / kUnitRows;
  s.check_units = (p + kUnitRows - 1) / kUnitRows;
  s.tile_units = s.data_units + s.check_units;
  if (g.prm.t % kSliceBytes != 0 || n > kMaxSmemRows || s.kpad + p > kMaxSmemSlots) return;
  auto slot = [&](int32_t m) -> uint16_t {
    return static_cast<uint16_t>(static_cast<uint32_t>(m) < k ? m : s.kpad + (m - k));
  };
  s.pre_slots.resize(g.pre_col.size());
  for (size_t e = 0; e < g.pre_col.size(); ++e) s.pre_slots[e] = slot(g.pre_col[e]);

  struct Item {
    bool split;
    uint32_t steps;                  // edge steps (the store step comes on top)
    uint32_t rows[4];
    std::vector<uint16_t> lanes[4];  // per group, the slots of its steps
  };
  std::vector<Item> items;
  std::vector<uint32_t> light;
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t d = static_cast<uint32_t>(g.lt_row_ptr[j + 1] - g.lt_row_ptr[j]);
    if (d > static_cast<uint32_t>(kSplitThreshold)) {
      Item it;
      it.split = true;
      it.rows[0] = it.rows[1] = it.rows[2] = it.rows[3] = j;
      for (uint32_t e = 0; e < d; ++e) it.lanes[e % 4].push_back(slot(g.lt_col[g.lt_row_ptr[j] + e]));
      it.steps = (d + 3) / 4;
      items.push_back(std::move(it));
    } else {
      light.push_back(j);
    }
  }
  std::stable_sort(light.begin(), light.end(), [&](uint32_t a, uint32_t b) {
    return (g.lt_row_ptr[a + 1] - g.lt_row_ptr[a]) > (g.lt_row_ptr[b + 1] - g.lt_row_ptr[b]);
  });
  for (size_t i = 0; i < light.size(); i += 4) {
    Item it;
    it.split = false;
    it.steps = 0;
    for (int q = 0; q < 4; ++q) {
      if (i + q < light.size()) {
        const uint32_t j = light[i + q];
        it.rows[q] = j;
        for (int32_t e = g.lt_row_ptr[j]; e < g.lt_row_ptr[j + 1]; ++e) it.lanes[q].push_back(slot(g.lt_col[e]));
        it.steps = std::max<uint32_t>(it.steps, static_cast<uint32_t>(it.lanes[q].size()));
      } else {
        it.rows[q] = UINT32_MAX;
      }
    }
    items.push_back(std::move(it));
  }
  // LPT over warps; cost = edge steps + the store step (+1 for the split shuffles)
  auto cost = [](const Item &it) { return it.steps + (it.split ? 2u : 1u); };
  std::vector<uint32_t> order(items.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cost(items[a]) > cost(items[b]); });
  using Load = std::pair<uint64_t, int>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int w = 0; w < kConsumerWarps; ++w) heap.push({0, w});
  std::vector<std::vector<uint32_t>> per_warp(kConsumerWarps);
  for (uint32_t idx : order) {
    Load l = heap.top();
    heap.pop();
    per_warp[l.second].push_back(idx);
    heap.push({l.first + cost(items[idx]), l.second});
  }
  // per-warp step streams: [steps x 4 values] per item, then its store step
  std::vector<std::vector<uint16_t>> streams(kConsumerWarps);
  s.warp_steps.assign(kConsumerWarps, 0);
  s.steps_max = s.steps_total = 0;
  for (int w = 0; w < kConsumerWarps; ++w) {
    std::vector<uint16_t> &st = streams[w];
    for (uint32_t idx : per_warp[w]) {
      const Item &it = items[idx];
      for (uint32_t e = 0; e < it.steps; ++e)
        for (int q = 0; q < 4; ++q) st.push_back(e < it.lanes[q].size() ? it.lanes[q][e] : kIdle);
      for (int q = 0; q < 4; ++q) {
        uint16_t v;
        if (it.split) v = static_cast<uint16_t>(kStoreFlag | kSplitFlag | it.rows[0]);
        else if (it.rows[q] == UINT32_MAX) v = kStoreNone;
        else v = static_cast<uint16_t>(kStoreFlag | it.rows[q]);
        st.push_back(v);
      }
    }
    s.warp_steps[w] = static_cast<uint32_t>(st.size() / 4);
    s.steps_max = std::max(s.steps_max, s.warp_steps[w]);
    s.steps_total += s.warp_steps[w];
  }
  if (s.steps_max > kMaxWarpSteps) return;  // too much work per tile for the register schedule
  s.regs = s.steps_max <= 16u * kStepsPerReg ? 16 : kSchedRegsMax;
  // word layout per warp: word (r*32 + lane) = register r of lane `lane`; step e, group q is
  // the (q&1) half of stream word 2e + (q>>1) -> register (2e+(q>>1))/32, lane (2e+(q>>1))%32
  const uint32_t wpw = s.regs * 32;
  s.words.assign(static_cast<size_t>(kConsumerWarps) * wpw, (static_cast<uint32_t>(kIdle) << 16) | kIdle);
  for (int w = 0; w < kConsumerWarps; ++w) {
    const std::vector<uint16_t> &st = streams[w];
    for (size_t e = 0; e < st.size() / 4; ++e)
      for (int q = 0; q < 4; ++q) {
        const uint32_t word = static_cast<uint32_t>(2 * e + (q >> 1));
        uint32_t &dst = s.words[static_cast<size_t>(w) * wpw + word];
        const uint32_t v = st[e * 4 + q];
        dst = (q & 1) ? ((dst & 0x0000FFFFu) | (v << 16)) : ((dst & 0xFFFF0000u) | v);
      }
  }
  g.smem_eligible = true;
}

}  // namespace fsb
