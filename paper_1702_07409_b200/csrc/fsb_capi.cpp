// C ABI of libfsb200.so (include/fsb.h): argument validation, ownership, error reporting.
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "fsb_internal.h"

namespace fsb {
namespace {
thread_local std::string g_err;
thread_local uint32_t g_launches = 0;
}  // namespace
void set_error(const std::string &msg) { g_err = msg; }
}  // namespace fsb

using fsb::set_error;

namespace {

fs_status finish_create(fs_graph *h, uint32_t flags, fs_graph **out) {
  fsb::Graph &g = h->g;
  fs_status lv = fsb::build_precode_levels(g);
  if (lv != FS_OK) {
    delete h;
    return lv;
  }
  fsb::build_smem_schedule(g);
  {  // fixed-size edge windows of the GLOBAL LT kernel (FSB_WIN_ROWS: rows per window, 0 = none;
     // FSB_WIN_REGS: 32-edge registers per lane, 3..5)
    static const uint32_t win_rows = [] {
      const char *e = std::getenv("FSB_WIN_ROWS");
      return e ? static_cast<uint32_t>(std::atoi(e)) : fsb::kWinRows;
    }();
    static const uint32_t win_regs = [] {
      const char *e = std::getenv("FSB_WIN_REGS");
      const uint32_t r = e ? static_cast<uint32_t>(std::atoi(e)) : fsb::kWinRegs;
      return r < 3 ? 3u : (r > 5 ? 5u : r);
    }();
    fsb::build_lt_windows(g, win_rows, win_regs);
  }
  if (!(flags & FS_GRAPH_HOST_ONLY)) {
    fs_status st = fsb::upload_graph(g);
    if (st != FS_OK) {
      fsb::free_device(g);
      delete h;
      return st;
    }
  } else {
    g.dev.device = -1;
  }
  *out = h;
  return FS_OK;
}

fs_graph *new_graph(const fs_params *prm) {
  fs_graph *h = new (std::nothrow) fs_graph();
  if (!h) return nullptr;
  fsb::Graph &g = h->g;
  g.prm = *prm;
  if (prm->dist == FS_DIST_FINITE && prm->fin_len && prm->fin_deg && prm->fin_prob) {
    g.fin_deg.assign(prm->fin_deg, prm->fin_deg + prm->fin_len);
    g.fin_prob.assign(prm->fin_prob, prm->fin_prob + prm->fin_len);
    g.prm.fin_deg = g.fin_deg.data();
    g.prm.fin_prob = g.fin_prob.data();
  } else {
    g.prm.fin_deg = nullptr;
    g.prm.fin_prob = nullptr;
    g.prm.fin_len = 0;
  }
  return h;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

fs_status fs_graph_create(const fs_params *prm, uint32_t flags, fs_graph **out) {
  fsb::set_error("");
  if (!prm || !out) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  fs_status st = fsb::validate_params(*prm);
  if (st != FS_OK) return st;
  fs_graph *h = new_graph(prm);
  if (!h) { set_error("out of host memory"); return FS_ENOMEM; }
  try {
    st = fsb::generate_csr(h->g);
  } catch (const std::bad_alloc &) {
    st = FS_ENOMEM;
    set_error("out of host memory");
  }
  if (st != FS_OK) {
    delete h;
    return st;
  }
  return finish_create(h, flags, out);
}

fs_status fs_graph_from_csr(const fs_params *prm, const int32_t *pre_row_ptr, const int32_t *pre_col,
                            const int32_t *lt_row_ptr, const int32_t *lt_col, uint32_t flags, fs_graph **out) {
  fsb::set_error("");
  if (!prm || !out || !lt_row_ptr || !lt_col) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  fs_status st = fsb::validate_params(*prm);
  if (st != FS_OK) return st;
  if (prm->p > 0 && (!pre_row_ptr || !pre_col)) { set_error("precode CSR missing"); return FS_EINVAL; }
  fs_graph *h = new_graph(prm);
  if (!h) { set_error("out of host memory"); return FS_ENOMEM; }
  fsb::Graph &g = h->g;
  const uint32_t p = prm->p, n = prm->n;
  if (p) {
    g.pre_row_ptr.assign(pre_row_ptr, pre_row_ptr + p + 1);
    if (g.pre_row_ptr[p] < 0) { delete h; set_error("invalid precode CSR"); return FS_EINVAL; }
    g.pre_col.assign(pre_col, pre_col + g.pre_row_ptr[p]);
    if (g.prm.precode == FS_PRECODE_ARRAY) g.prm.d_p = static_cast<uint32_t>(g.pre_row_ptr[1] - g.pre_row_ptr[0]);
  } else {
    g.pre_row_ptr.assign(1, 0);
  }
  g.lt_row_ptr.assign(lt_row_ptr, lt_row_ptr + n + 1);
  if (g.lt_row_ptr[n] < 0) { delete h; set_error("invalid LT CSR"); return FS_EINVAL; }
  g.lt_col.assign(lt_col, lt_col + g.lt_row_ptr[n]);
  st = fsb::validate_csr(g);
  if (st != FS_OK) {
    delete h;
    return st;
  }
  g.max_degree = 0;
  for (uint32_t j = 0; j < n; ++j)
    g.max_degree = std::max<uint32_t>(g.max_degree, static_cast<uint32_t>(g.lt_row_ptr[j + 1] - g.lt_row_ptr[j]));
  return finish_create(h, flags, out);
}

fs_status fs_graph_csr(const fs_graph *h, const int32_t **pre_row_ptr, const int32_t **pre_col,
                       const int32_t **lt_row_ptr, const int32_t **lt_col, uint64_t *lt_nnz) {
  if (!h) { set_error("null graph"); return FS_EINVAL; }
  const fsb::Graph &g = h->g;
  if (pre_row_ptr) *pre_row_ptr = g.pre_row_ptr.data();
  if (pre_col) *pre_col = g.pre_col.empty() ? nullptr : g.pre_col.data();
  if (lt_row_ptr) *lt_row_ptr = g.lt_row_ptr.data();
  if (lt_col) *lt_col = g.lt_col.data();
  if (lt_nnz) *lt_nnz = g.lt_col.size();
  return FS_OK;
}

fs_status fs_graph_get_info(const fs_graph *h, fs_graph_info *info) {
  if (!h || !info) { set_error("null argument"); return FS_EINVAL; }
  const fsb::Graph &g = h->g;
  std::memset(info, 0, sizeof(*info));
  info->k = g.prm.k;
  info->p = g.prm.p;
  info->d_p = g.prm.d_p;
  info->n = g.prm.n;
  info->t = g.prm.t;
  info->lt_nnz = g.lt_col.size();
  info->pre_nnz = g.pre_col.size();
  info->max_degree = g.max_degree;
  info->variant = g.variant;
  info->smem_eligible = g.smem_eligible ? 1 : 0;
  info->smem_bytes = g.smem_bytes;
  info->sched_bytes = static_cast<uint32_t>(g.sched.words.size() * 4);
  info->sched_steps_max = g.sched.steps_max;
  info->sched_steps_avg = (g.sched.steps_total + g.sched.nconsumer / 2) / std::max<uint32_t>(g.sched.nconsumer, 1);
  info->device = g.dev.device;
  info->lt_windows = g.win.count;
  return FS_OK;
}

fs_status fs_graph_set_variant(fs_graph *h, int32_t variant) {
  if (!h) { set_error("null graph"); return FS_EINVAL; }
  if (variant != FS_VARIANT_AUTO && variant != FS_VARIANT_SMEM && variant != FS_VARIANT_GLOBAL) {
    set_error("unknown variant");
    return FS_EINVAL;
  }
  if (variant == FS_VARIANT_SMEM && !h->g.smem_eligible) {
    set_error("SMEM variant not eligible for this graph");
    return FS_EUNSUPPORTED;
  }
  h->g.variant = variant;
  return FS_OK;
}

static fs_status check_device_graph(const fs_graph *h) {
  if (!h) { set_error("null graph"); return FS_EINVAL; }
  if (h->g.dev.device < 0) { set_error("host-only graph has no device copy"); return FS_EUNSUPPORTED; }
  return FS_OK;
}

fs_status fs_encode_range(const fs_graph *h, const uint8_t *d_data, uint8_t *d_checks, uint8_t *d_coded,
                          uint32_t row_begin, uint32_t row_end, uint64_t col_begin, uint64_t col_end, void *stream) {
  fsb::set_error("");
  fsb::g_launches = 0;
  fs_status st = check_device_graph(h);
  if (st != FS_OK) return st;
  const fsb::Graph &g = h->g;
  if (row_begin > row_end || row_end > g.prm.n) { set_error("invalid row range"); return FS_EINVAL; }
  if (col_begin > col_end || col_end > g.prm.t || col_begin % 16 || col_end % 16) {
    set_error("invalid column range: need col_begin <= col_end <= t, multiples of 16");
    return FS_EINVAL;
  }
  if (!d_data || !aligned16(d_data)) { set_error("d_data must be a 16-B aligned device pointer"); return FS_EINVAL; }
  if (g.prm.p > 0 && (!d_checks || !aligned16(d_checks))) { set_error("d_checks must be 16-B aligned, non-NULL when p > 0"); return FS_EINVAL; }
  if (g.prm.p == 0 && d_checks) { set_error("d_checks must be NULL when p == 0"); return FS_EINVAL; }
  if (row_end > row_begin && (!d_coded || !aligned16(d_coded))) { set_error("d_coded must be a 16-B aligned device pointer"); return FS_EINVAL; }
  if (col_end == col_begin) return FS_OK;
  const uint64_t t = g.prm.t;
  uint32_t launches = 0;
  st = fsb::launch_encode(g, 1, d_data, g.prm.k * t, d_checks, g.prm.p * t, d_coded,
                          static_cast<uint64_t>(row_end - row_begin) * t, row_begin, row_end, col_begin, col_end,
                          stream, &launches);
  if (st == FS_OK) fsb::g_launches = launches;
  return st;
}

fs_status fs_encode(const fs_graph *h, const uint8_t *d_data, uint8_t *d_checks, uint8_t *d_coded,
                    uint32_t row_begin, uint32_t row_end, void *stream) {
  if (!h) { fsb::set_error("null graph"); fsb::g_launches = 0; return FS_EINVAL; }
  return fs_encode_range(h, d_data, d_checks, d_coded, row_begin, row_end, 0, h->g.prm.t, stream);
}

fs_status fs_encode_stripes(const fs_graph *h, uint32_t S, const uint8_t *d_data, uint64_t data_stride,
                            uint8_t *d_checks, uint64_t checks_stride, uint8_t *d_coded, uint64_t coded_stride,
                            void *stream) {
  fsb::set_error("");
  fsb::g_launches = 0;
  fs_status st = check_device_graph(h);
  if (st != FS_OK) return st;
  const fsb::Graph &g = h->g;
  if (S == 0) return FS_OK;
  const uint64_t t = g.prm.t;
  if (!d_data || !aligned16(d_data) || data_stride < g.prm.k * t || data_stride % 16) {
    set_error("d_data must be 16-B aligned with data_stride >= k*t, a multiple of 16");
    return FS_EINVAL;
  }
  if (g.prm.p > 0 && (!d_checks || !aligned16(d_checks) || checks_stride < g.prm.p * t || checks_stride % 16)) {
    set_error("d_checks must be 16-B aligned with checks_stride >= p*t, a multiple of 16");
    return FS_EINVAL;
  }
  if (g.prm.p == 0 && d_checks) { set_error("d_checks must be NULL when p == 0"); return FS_EINVAL; }
  if (!d_coded || !aligned16(d_coded) || coded_stride < g.prm.n * t || coded_stride % 16) {
    set_error("d_coded must be 16-B aligned with coded_stride >= n*t, a multiple of 16");
    return FS_EINVAL;
  }
  uint32_t launches = 0;
  st = fsb::launch_encode(g, S, d_data, data_stride, d_checks, checks_stride, d_coded, coded_stride, 0, g.prm.n, 0,
                          g.prm.t, stream, &launches);
  if (st == FS_OK) fsb::g_launches = launches;
  return st;
}

fs_status fs_encode_host(const fs_graph *h, uint32_t S, const uint8_t *h_data, uint64_t data_stride,
                         uint8_t *h_checks, uint64_t checks_stride, uint8_t *h_coded, uint64_t coded_stride,
                         uint32_t chunks, void *stream) {
  fsb::set_error("");
  fsb::g_launches = 0;
  fs_status st = check_device_graph(h);
  if (st != FS_OK) return st;
  const fsb::Graph &g = h->g;
  if (S == 0) return FS_OK;
  const uint64_t t = g.prm.t, k = g.prm.k, p = g.prm.p, n = g.prm.n;
  if (S == 1) {  // one stripe: symbols contiguous (the column chunks are strided by t)
    data_stride = std::max(data_stride, k * t);
    checks_stride = std::max(checks_stride, p * t);
    coded_stride = std::max(coded_stride, n * t);
  }
  if (!h_data || data_stride < k * t) { set_error("h_data must be non-NULL with data_stride >= k*t"); return FS_EINVAL; }
  if (p > 0 && (!h_checks || checks_stride < p * t)) {
    set_error("h_checks must be non-NULL with checks_stride >= p*t when p > 0");
    return FS_EINVAL;
  }
  if (p == 0 && h_checks) { set_error("h_checks must be NULL when p == 0"); return FS_EINVAL; }
  if (!h_coded || coded_stride < n * t) { set_error("h_coded must be non-NULL with coded_stride >= n*t"); return FS_EINVAL; }
  {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g.dev.device) {
      set_error("the graph lives on device " + std::to_string(g.dev.device) + ", the current device is " +
                std::to_string(cur));
      return FS_EINVAL;
    }
  }
  fs_graph *hm = const_cast<fs_graph *>(h);  // the staging cache is the graph's, not its contents
  std::lock_guard<std::mutex> lock(hm->io_mu);
  if (!hm->io) hm->io.reset(new (std::nothrow) fsb::IoCache());
  if (!hm->io) { set_error("out of host memory"); return FS_ENOMEM; }
  uint32_t launches = 0;
  st = fsb::encode_host(g, *hm->io, S, h_data, data_stride, h_checks, checks_stride, h_coded, coded_stride,
                        chunks ? chunks : 32u, stream, &launches);
  if (st == FS_OK) fsb::g_launches = launches;
  return st;
}

fs_status fs_graph_schedule(const fs_graph *h, const uint32_t **words, uint64_t *nwords, uint32_t *cont_base,
                            const uint32_t **warp_info, uint32_t *nwarps, uint32_t *kpad, uint32_t *zero_even) {
  if (!h) { set_error("null graph"); return FS_EINVAL; }
  const fsb::Graph &g = h->g;
  if (!g.smem_eligible || g.sched.words.empty()) { set_error("graph has no SMEM schedule"); return FS_EUNSUPPORTED; }
  if (words) *words = g.sched.words.data();
  if (nwords) *nwords = g.sched.words.size();
  if (cont_base) *cont_base = g.sched.cont_base;
  if (warp_info) *warp_info = g.sched.warp_info.data();
  if (nwarps) *nwarps = g.sched.nconsumer;
  if (kpad) *kpad = g.sched.kpad;
  if (zero_even) *zero_even = g.sched.zero_even;
  return FS_OK;
}

fs_status fs_graph_windows(const fs_graph *h, const uint32_t **hdr, const uint32_t **ent, uint32_t *count,
                           uint32_t *entries) {
  if (!h) { set_error("null graph"); return FS_EINVAL; }
  const fsb::Graph &g = h->g;
  if (!g.win.count) { set_error("graph has no LT edge windows"); return FS_EUNSUPPORTED; }
  if (hdr) *hdr = g.win.hdr.data();
  if (ent) *ent = g.win.ent.data();
  if (count) *count = g.win.count;
  if (entries) *entries = g.win.entries;
  return FS_OK;
}

fs_status fs_debug_counters(uint64_t *out, uint32_t n) {
  if (!out) { set_error("null argument"); return FS_EINVAL; }
  return fsb::read_debug_counters(out, n);
}

fs_status fs_decode_plan_create(const fs_graph *h, const uint8_t *received, uint32_t flags, fs_decode_plan **out) {
  fsb::set_error("");
  if (!h || !received || !out) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  if (flags & ~(FS_GRAPH_HOST_ONLY | FS_DECODE_ELIMINATE)) { set_error("unknown decode flags"); return FS_EINVAL; }
  fs_decode_plan *d = new (std::nothrow) fs_decode_plan();
  if (!d) { set_error("out of host memory"); return FS_ENOMEM; }
  fs_status st;
  try {
    st = fsb::build_decode_plan(h->g, received, d->pl, (flags & FS_DECODE_ELIMINATE) != 0);
  } catch (const std::bad_alloc &) {
    st = FS_ENOMEM;
    set_error("out of host memory");
  }
  if (st == FS_OK && !(flags & FS_GRAPH_HOST_ONLY)) st = fsb::upload_decode_plan(d->pl);
  if (st != FS_OK) {
    fsb::free_decode_plan(d->pl);
    delete d;
    return st;
  }
  *out = d;
  return FS_OK;
}

fs_status fs_decode_plan_info(const fs_decode_plan *d, fs_decode_info *info) {
  if (!d || !info) { set_error("null argument"); return FS_EINVAL; }
  const fsb::DecodePlan &pl = d->pl;
  std::memset(info, 0, sizeof(*info));
  info->K = pl.K;
  info->n = pl.n;
  info->received = pl.received;
  info->levels = static_cast<uint32_t>(pl.level_ptr.size() - 1);
  info->rows = static_cast<uint32_t>(pl.target.size());
  for (uint32_t m = 0; m < pl.K; ++m) {
    info->recovered += pl.state[m] ? 1 : 0;
    if (m < pl.k) info->recovered_data += pl.state[m] ? 1 : 0;
  }
  for (size_t L = 0; L + 1 < pl.level_ptr.size(); ++L)
    info->max_level_rows = std::max<uint32_t>(info->max_level_rows, pl.level_ptr[L + 1] - pl.level_ptr[L]);
  info->xor_sources = pl.src.size();
  info->eliminated = pl.eliminated;
  info->elim_skipped = pl.elim_skipped;
  info->inactivated = pl.inactivated;
  info->work_rows = pl.work_rows;
  return FS_OK;
}

fs_status fs_decode_plan_state(const fs_decode_plan *d, const uint8_t **state, const int32_t **level_of) {
  if (!d) { set_error("null argument"); return FS_EINVAL; }
  if (state) *state = d->pl.state.data();
  if (level_of) *level_of = d->pl.level_of.data();
  return FS_OK;
}

fs_status fs_decode(const fs_decode_plan *d, uint32_t S, const uint8_t *d_coded, uint64_t coded_stride,
                    uint8_t *d_inter, uint64_t inter_stride, void *stream) {
  fsb::set_error("");
  fsb::g_launches = 0;
  if (!d) { set_error("null plan"); return FS_EINVAL; }
  const fsb::DecodePlan &pl = d->pl;
  if (pl.device < 0) { set_error("host-only plan has no device copy"); return FS_EUNSUPPORTED; }
  if (S == 0) return FS_OK;
  if (!d_coded || !aligned16(d_coded) || coded_stride < pl.n * pl.t || coded_stride % 16) {
    set_error("d_coded must be 16-B aligned with coded_stride >= n*t, a multiple of 16");
    return FS_EINVAL;
  }
  if (!d_inter || !aligned16(d_inter) || inter_stride < static_cast<uint64_t>(pl.K) * pl.t || inter_stride % 16) {
    set_error("d_inter must be 16-B aligned with inter_stride >= (k+p)*t, a multiple of 16");
    return FS_EINVAL;
  }
  uint32_t launches = 0;
  fs_status st = fsb::launch_decode(pl, S, d_coded, coded_stride, d_inter, inter_stride, stream, &launches);
  if (st == FS_OK) fsb::g_launches = launches;
  return st;
}

void fs_decode_plan_free(fs_decode_plan *d) {
  if (!d) return;
  fsb::free_decode_plan(d->pl);
  delete d;
}

// ------------------------------------------------------------ repair / update (NEXT-3)
fs_status fs_checks_create(const fs_graph *h, uint32_t flags, fs_checks **out) {
  fsb::set_error("");
  if (!h || !out) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  if (flags & ~(FS_CHECKS_M1 | FS_CHECKS_M2)) { set_error("unknown check flags"); return FS_EINVAL; }
  fs_checks *c = new (std::nothrow) fs_checks();
  if (!c) { set_error("out of host memory"); return FS_ENOMEM; }
  fs_status st;
  try {
    st = fsb::build_check_data(h->g, flags, c->cd);
  } catch (const std::bad_alloc &) {
    st = FS_ENOMEM;
    set_error("out of host memory");
  }
  if (st != FS_OK) {
    delete c;
    return st;
  }
  c->n = h->g.prm.n;
  c->K = h->g.prm.k + h->g.prm.p;
  *out = c;
  return FS_OK;
}

fs_status fs_checks_from_data(const fs_graph *h, const int32_t *data, uint64_t len, fs_checks **out) {
  fsb::set_error("");
  if (!h || !out || (len && !data)) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  fs_checks *c = new (std::nothrow) fs_checks();
  if (!c) { set_error("out of host memory"); return FS_ENOMEM; }
  fs_status st = fsb::parse_check_data(h->g, data, len, c->cd);
  if (st != FS_OK) {
    delete c;
    return st;
  }
  c->n = h->g.prm.n;
  c->K = h->g.prm.k + h->g.prm.p;
  *out = c;
  return FS_OK;
}

fs_status fs_checks_data(const fs_checks *c, const int32_t **data, uint64_t *len) {
  if (!c) { set_error("null argument"); return FS_EINVAL; }
  if (data) *data = c->cd.data.empty() ? nullptr : c->cd.data.data();
  if (len) *len = c->cd.data.size();
  return FS_OK;
}

fs_status fs_checks_info_get(const fs_checks *c, fs_checks_info *info) {
  if (!c || !info) { set_error("null argument"); return FS_EINVAL; }
  std::memset(info, 0, sizeof(*info));
  info->sweeps = c->cd.sweeps;
  info->zero_columns = c->cd.zero_columns;
  info->weight1_columns = c->cd.weight1_columns;
  info->group2 = c->cd.group2;
  info->group3 = c->cd.group3;
  info->derived = c->cd.derived;
  info->len = c->cd.data.size();
  return FS_OK;
}

void fs_checks_free(fs_checks *c) { delete c; }

fs_status fs_repair_plan_create(const fs_graph *h, const fs_checks *c, const uint8_t *erased, const uint32_t *want,
                                uint32_t nwant, uint32_t flags, fs_repair_plan **out) {
  fsb::set_error("");
  if (!h || !c || !erased || !out || (nwant && !want)) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  if (c->n > h->g.prm.n || c->K != h->g.prm.k + h->g.prm.p) {
    set_error("check data does not fit the graph (needs the same K and n_checks <= n)");
    return FS_EINVAL;
  }
  fs_repair_plan *r = new (std::nothrow) fs_repair_plan();
  if (!r) { set_error("out of host memory"); return FS_ENOMEM; }
  fs_status st;
  try {
    st = fsb::build_repair_plan(h->g, c->cd, erased, want, nwant, r->pl, r->rs);
  } catch (const std::bad_alloc &) {
    st = FS_ENOMEM;
    set_error("out of host memory");
  }
  if (st == FS_OK && !(flags & FS_GRAPH_HOST_ONLY)) st = fsb::upload_decode_plan(r->pl);
  if (st != FS_OK) {
    fsb::free_decode_plan(r->pl);
    delete r;
    return st;
  }
  *out = r;
  return FS_OK;
}

fs_status fs_repair_plan_info(const fs_repair_plan *r, fs_repair_info *info) {
  if (!r || !info) { set_error("null argument"); return FS_EINVAL; }
  std::memset(info, 0, sizeof(*info));
  info->erased = r->rs.erased;
  info->repaired = r->rs.repaired;
  info->unrepaired = r->rs.unrepaired;
  info->want_missing = r->rs.want_missing;
  info->levels = r->rs.levels;
  info->rows = r->rs.rows;
  info->xor_sources = r->rs.xor_sources;
  return FS_OK;
}

fs_status fs_repair_plan_rows(const fs_repair_plan *r, const uint32_t **level_ptr, uint32_t *levels,
                              const int32_t **target, const int32_t **src_ptr, const uint32_t **src) {
  if (!r) { set_error("null argument"); return FS_EINVAL; }
  const fsb::DecodePlan &pl = r->pl;
  if (level_ptr) *level_ptr = pl.level_ptr.data();
  if (levels) *levels = static_cast<uint32_t>(pl.level_ptr.size() - 1);
  if (target) *target = pl.target.empty() ? nullptr : pl.target.data();
  if (src_ptr) *src_ptr = pl.src_ptr.data();
  if (src) *src = pl.src.empty() ? nullptr : pl.src.data();
  return FS_OK;
}

fs_status fs_repair(const fs_repair_plan *r, uint32_t S, uint8_t *d_coded, uint64_t coded_stride, uint8_t *d_inter,
                    uint64_t inter_stride, void *stream) {
  fsb::set_error("");
  fsb::g_launches = 0;
  if (!r) { set_error("null plan"); return FS_EINVAL; }
  const fsb::DecodePlan &pl = r->pl;
  if (pl.device < 0) { set_error("host-only plan has no device copy"); return FS_EUNSUPPORTED; }
  if (S == 0 || pl.target.empty()) return FS_OK;
  if (!d_coded || !aligned16(d_coded) || coded_stride < pl.n * pl.t || coded_stride % 16) {
    set_error("d_coded must be 16-B aligned with coded_stride >= n*t, a multiple of 16");
    return FS_EINVAL;
  }
  bool wants = false;
  for (int32_t tg : pl.target) wants = wants || !(static_cast<uint32_t>(tg) & fsb::kSrcCoded);
  if (wants && (!d_inter || !aligned16(d_inter) || inter_stride < static_cast<uint64_t>(pl.K) * pl.t ||
                inter_stride % 16)) {
    set_error("d_inter must be 16-B aligned with inter_stride >= (k+p)*t when the plan reads symbols");
    return FS_EINVAL;
  }
  uint32_t launches = 0;
  fs_status st = fsb::launch_plan(pl, S, d_coded, coded_stride, d_inter, inter_stride, stream, &launches);
  if (st == FS_OK) fsb::g_launches = launches;
  return st;
}

void fs_repair_plan_free(fs_repair_plan *r) {
  if (!r) return;
  fsb::free_decode_plan(r->pl);
  delete r;
}

fs_status fs_graph_extend(const fs_graph *h, uint32_t extra_files, uint32_t flags, fs_graph **out) {
  fsb::set_error("");
  if (!h || !out) { set_error("null argument"); return FS_EINVAL; }
  *out = nullptr;
  if (extra_files == 0) { set_error("extra_files must be >= 1"); return FS_EINVAL; }
  fs_params prm = h->g.prm;  // fin_* point into h's vectors; fs_graph_create copies them
  const uint32_t s = std::max<uint32_t>(prm.files, 1);
  const uint64_t n2 = static_cast<uint64_t>(prm.n) + static_cast<uint64_t>(extra_files) * (prm.n / s);
  if (n2 >= (1ull << 31) || static_cast<uint64_t>(s) + extra_files >= (1ull << 31)) {
    set_error("extended n too large");
    return FS_EINVAL;
  }
  prm.n = static_cast<uint32_t>(n2);
  prm.files = s + extra_files;
  return fs_graph_create(&prm, flags, out);
}

uint32_t fs_last_launch_count(void) { return fsb::g_launches; }

void fs_free(fs_graph *h) {
  if (!h) return;
  h->io.reset();  // synchronises the fs_encode_host streams before the graph's device memory goes
  fsb::free_device(h->g);
  delete h;
}

const char *fs_last_error(void) { return fsb::g_err.c_str(); }

const char *fs_version(void) { return "fsb200 0.1.0 (sm_100a)"; }

}  // extern "C"
