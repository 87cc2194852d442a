// Internal declarations of libfsb200 (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fsb.h"

namespace fsb {

// ----------------------------------------------------------------- SMEM kernel geometry
// A tile = (stripe, 64-byte slice of every symbol): its K intermediate rows, 64 B each, staged
// in shared memory in units of kUnitRows rows (one TMA box of kUnitRows x 64 B).  Two tile
// buffers (double buffering) plus the per-tile LT schedule fit in shared memory.
constexpr int kSliceBytes = 64;
constexpr int kUnitRows = 64;
constexpr int kUnitBytes = kUnitRows * kSliceBytes;     // 4 KiB
constexpr int kConsumerWarps = 24;
constexpr int kHalvesPerWarp = 8;                        // precode half-groups: 4 lanes x 16 B = 64 B
constexpr int kGroupsPerWarp = 16;                       // LT groups: 2 lanes x 32 B = 64 B
constexpr int kPrecodeWarps = 3;                         // precode (a3) warps per CTA
constexpr int kThreads = (kConsumerWarps + 1 + kPrecodeWarps) * 32;  // + 1 TMA warp
constexpr int kSplitThreshold = 60;                      // rows of degree > this are split:
constexpr int kSplit2Max = 120;                           //   over the 2 halves of a group (<= this)
                                                         //   or over the 8 half-groups of a warp

// LT work is done by *groups* of 2 lanes, 16 per warp: group g = lanes 2g, 2g+1; lane l2 = lane & 1
// owns the 32 contiguous bytes 32*l2 .. 32*l2+31 of a 64-B row slice and reads them with two
// 128-bit shared loads per slot (pieces 2*l2+s and 2*l2+1-s, s = g & 1).
// Bank rule: a 128-bit shared load is served in phases of 8 lanes = groups 4m..4m+3.  A 64-B row r
// occupies the 16 banks of half (r & 1) of a 128-B line; the two groups of a phase with the same s
// read two different 16-B pieces of their rows per load, so the phase is conflict-free iff groups
// g and g^2 read rows of opposite parity (then the 8 lanes cover 8 distinct 16-B bank quads).  The
// host schedule guarantees it in every step: a *pair* of rows sits in groups (g, g^2) -- pair q
// in groups 4(q>>1) + (q&1) (half 0) and that + 2 (half 1) -- and half 0 reads an even row exactly
// when half 1 reads an odd row (padding uses the even / odd zero rows).  Against 16-B lanes (4 per
// row) one schedule load feeds twice the gathers and a warp's item carries 16 rows instead of 8
// (tools/microbench/mb15.cu variant 5: 4.15 clk per gather vs 4.29).
//
// Item-record schedule.  A warp's per-tile LT work is a list of *items*; an item gives each of
// the warp's 16 groups one output row and the same number L of source slots.  A slot is an
// 11-bit tile row (data m -> m, check i -> kpad+i, padding -> zero_even / zero_odd); two slots
// share a 32-bit word as  a | b << 21  (bits 11..20 zero; bits 11..14 may carry flags, which the
// address arithmetic ignores), so the kernel forms the shared address of `b` with one shift-add
// (sbase + (w >> 15)).  Two streams, copied into shared memory once per CTA, in 256-byte chunks
// (16 groups x 16 B; group g's 16 B at uint4 index chunk*16 + g):
//   heads: one chunk per item: word 0 = row | ctrl << 16, words 1..3 = slots 0..5; ctrl =
//          L | pair-split << 14 | warp-split << 15 (identical in all 16 groups); row =
//          kNoRow for a group that stores nothing; word 1 bit 11 (kPairFlag) marks a
//          group whose partner half holds the other part of the same row;
//   conts: slots 6.. of items with L > 6, 8 per chunk (4 words), items in the same order.
// Heavy rows: degree <= kSplit2Max -> a pair-split: evens in half 0, odds in half 1 of one pair
// (combined by one xor-4 warp shuffle, stored by half 0); larger -> a warp-split item: evens over
// the eight half-0, odds over the eight half-1 groups (four warp shuffles, same row in all 16).
constexpr uint32_t kHeadSlots = 6;          // slots in an item's head chunk
constexpr uint32_t kChunkSlots = 8;         // slots in a continuation chunk
constexpr uint32_t kChunkBytes = kGroupsPerWarp * 16;
constexpr uint32_t kStreamPad = 2;          // zero chunks after each stream (prefetch overrun)
constexpr uint32_t kSlotBits = 11;
constexpr uint32_t kSlotHiShift = 21;
constexpr uint16_t kNoRow = 0xFFFF;
constexpr uint16_t kSplitBit = 0x8000;       // ctrl: warp-split item
constexpr uint16_t kPairSplitBit = 0x4000;   // ctrl: the item holds pair-split groups
constexpr uint32_t kPairFlag = 1u << 11;     // head word 1: this half-group's pair is split
constexpr uint32_t kMaxItemLen = 0x3FFF;
constexpr uint32_t kMaxSmemRows = 0xFFFE;   // n limit of the SMEM variant (16-bit output rows)
constexpr uint32_t kMaxSmemSlots = (1u << kSlotBits) - 1;  // tile rows (data + checks + zero rows)

// Host-built LT work schedule of the SMEM kernel (identical for every tile; fsb_graph.cpp).
struct SmemSchedule {
  std::vector<uint32_t> words;          // heads stream (+pad) then conts stream (+pad), uint32 words
  uint32_t cont_base = 0;               // first chunk of the conts stream in `words`
  std::vector<uint32_t> warp_info;      // nconsumer x {items, head_off, cont_off} (chunks)
  uint32_t nconsumer = kConsumerWarps;  // consumer warps; the other kConsumerWarps + kPrecodeWarps
                                        // - nconsumer warps (besides the TMA warp) run the precode
  std::vector<uint16_t> pre_slots;      // p * d_p data rows
  uint32_t kpad = 0;                    // data rows rounded up to kUnitRows
  uint32_t zero_even = 0;               // tile rows of the two all-zero padding rows
  uint32_t tile_rows = 0;               // rows of a tile buffer (zero_even + 2)
  uint32_t data_units = 0, tile_units = 0;
  uint32_t steps_max = 0, steps_total = 0;  // gather slots per half-group per warp: max, sum
  uint32_t pad_slots = 0;               // slots that read a zero row (parity / length padding)
};

// Fixed-size LT edge windows of the fsb_lt_win band kernel (built by build_lt_windows): window w
// holds whole rows [hdr[w].x, next window's first row), at most `rows` of them, as marked edges
// (bit 31 = last edge of a row) at ent[w * entries ...]; its edge count is padded to a multiple
// of 4 with kWinSkip entries at the start; hdr[w].y = the window's batches of 4.  entries =
// 32 x kWinRegs (one 32-bit register per lane per 32 edges).
constexpr uint32_t kWinRegs = 3;
constexpr uint32_t kWinRows = 12;
constexpr uint32_t kWinSkip = 1u << 30;
struct LtWindows {
  std::vector<uint32_t> hdr;   // 2 words per window: first row, batches of 4
  std::vector<uint32_t> ent;   // `entries` words per window
  uint32_t entries = 0;        // edge slots per window (32 x registers per lane)
  uint32_t count = 0;          // windows; 0 = some row does not fit a window (kernel not used)
};

struct DeviceBufs {
  int device = -1;
  int32_t *pre_row_ptr = nullptr, *pre_col = nullptr, *lt_row_ptr = nullptr, *lt_col = nullptr;
  uint32_t *lt_colf = nullptr;  // lt_col with bit 31 set on the last edge of each row
  uint32_t *win_hdr = nullptr, *win_ent = nullptr;  // LtWindows on the device
  uint32_t *sched = nullptr;
  uint32_t *warp_info = nullptr;
  uint16_t *pre_slots = nullptr;
  uint32_t *pre_level_ptr = nullptr;
};

struct Graph {
  fs_params prm{};
  std::vector<uint32_t> fin_deg;
  std::vector<double> fin_prob;
  std::vector<int32_t> pre_row_ptr, pre_col, lt_row_ptr, lt_col;
  std::vector<uint32_t> pre_level_ptr;  // precode levels: checks [lp[L], lp[L+1]) read checks < lp[L]
  uint32_t max_degree = 0;
  bool smem_eligible = false;
  SmemSchedule sched;
  LtWindows win;
  DeviceBufs dev;
  int32_t variant = FS_VARIANT_AUTO;
  int sm_count = 0;
  int smem_optin = 0;
  uint32_t smem_bytes = 0;   // dynamic smem of the SMEM kernel
};

// fsb_graph.cpp
fs_status validate_params(const fs_params &prm);
fs_status build_cdf(const fs_params &prm, std::vector<uint32_t> &deg, std::vector<double> &cdf);
fs_status generate_csr(Graph &g);
fs_status validate_csr(const Graph &g);
fs_status build_precode_levels(Graph &g);
void build_smem_schedule(Graph &g);
void build_lt_windows(Graph &g, uint32_t max_rows, uint32_t regs);

// fsb_kernels.cu
fs_status upload_graph(Graph &g);
void free_device(Graph &g);
fs_status launch_encode(const Graph &g, uint32_t S, const uint8_t *data, uint64_t data_stride,
                        uint8_t *checks, uint64_t checks_stride, uint8_t *coded,
                        uint64_t coded_stride, uint32_t row_begin, uint32_t row_end, uint64_t col_begin,
                        uint64_t col_end, void *stream, uint32_t *launches);

fs_status read_debug_counters(uint64_t *out, uint32_t n);

// fsb_capi.cpp
void set_error(const std::string &msg);

}  // namespace fsb

namespace fsb {
// staging of fs_encode_host (fsb_io.cpp): two library streams, their events, device buffers
struct IoCache {
  int device = -1;
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t start = nullptr, done[2] = {nullptr, nullptr};
  uint8_t *buf = nullptr;
  uint64_t bytes = 0;
  ~IoCache();
};
fs_status encode_host(const Graph &g, IoCache &c, uint32_t S, const uint8_t *h_data, uint64_t data_stride,
                      uint8_t *h_checks, uint64_t checks_stride, uint8_t *h_coded, uint64_t coded_stride,
                      uint32_t chunks, void *stream, uint32_t *launches);
}  // namespace fsb

struct fs_graph {
  fsb::Graph g;
  std::mutex io_mu;                        // fs_encode_host staging (created on first use)
  std::unique_ptr<fsb::IoCache> io;
};

// ------------------------------------------------------------------ decoder (NEXT-1, Alg 5)
namespace fsb {
// Decoding path of one (graph, received set): Alg 5 (DPG) levels over the received LT rows and
// the precode checks.  Row r of the plan recovers intermediate symbol target[r] as the XOR of
// its sources src[src_ptr[r] .. src_ptr[r+1]): an intermediate index m (recovered at an earlier
// level) or m | kSrcCoded for received coded row m; bit 31 (kSrcLast) marks a row's last source.
constexpr uint32_t kSrcCoded = 1u << 30;
constexpr uint32_t kSrcWork = 1u << 29;   // a workspace row (inactivation decoding, Z rows)
constexpr uint32_t kSrcIndex = kSrcWork - 1;
constexpr uint32_t kSrcLast = 1u << 31;
struct DecodePlan {
  uint32_t k = 0, p = 0, n = 0, K = 0;
  uint64_t t = 0;
  uint32_t received = 0;
  std::vector<uint32_t> level_ptr;   // levels+1 row offsets
  std::vector<int32_t> target;       // rows
  std::vector<int32_t> src_ptr;      // rows+1
  std::vector<uint32_t> src;         // flagged source list
  std::vector<uint8_t> state;        // K: 1 recovered, 0 not
  std::vector<int32_t> level_of;     // K: level that recovered it, -1
  uint32_t eliminated = 0;           // symbols of the final residual-elimination level
  uint32_t elim_skipped = 0;         // 1: residual too large, elimination not attempted
  uint32_t inactivated = 0;          // symbols inactivated by the completion phase
  uint32_t work_rows = 0;            // workspace rows (t bytes per stripe) the plan needs
  int device = -1;
  int32_t *d_target = nullptr, *d_src_ptr = nullptr;
  uint32_t *d_src = nullptr;
  int sm_count = 0;
  // the level launches captured once as a CUDA graph per (S, buffers, strides) and replayed
  // (fsb_kernels.cu; created by upload_decode_plan, guarded by its own mutex)
  std::shared_ptr<struct PlanGraphCache> gcache;
};
fs_status build_decode_plan(const Graph &g, const uint8_t *received, DecodePlan &pl, bool eliminate);
fs_status upload_decode_plan(DecodePlan &pl);
void free_decode_plan(DecodePlan &pl);
fs_status launch_decode(const DecodePlan &pl, uint32_t S, const uint8_t *coded, uint64_t coded_stride,
                        uint8_t *inter, uint64_t inter_stride, void *stream, uint32_t *launches);
// any plan (decode or repair): per-level fsb_dpg_level launches; repair targets write coded rows
fs_status launch_plan(const DecodePlan &pl, uint32_t S, uint8_t *coded, uint64_t coded_stride,
                      uint8_t *inter, uint64_t inter_stride, void *stream, uint32_t *launches);
}  // namespace fsb

struct fs_decode_plan {
  fsb::DecodePlan pl;
};

// ------------------------------------------------------------------ repair (NEXT-3, Alg 4)
namespace fsb {
struct CgaResult {
  std::vector<std::vector<int32_t>> b, l;  // final columns of B and L^{(2,3)}, ascending
  uint32_t sweeps = 0, zero_columns = 0, weight1_columns = 0;
  uint64_t updates = 0;
};
struct ChecksData {
  std::vector<int32_t> data;  // the <filename>_check.data integer array
  uint32_t sweeps = 0, zero_columns = 0, weight1_columns = 0, group2 = 0, group3 = 0, derived = 0;
};
struct RepairStats {
  uint32_t erased = 0, repaired = 0, unrepaired = 0, want_missing = 0, levels = 0, rows = 0;
  uint64_t xor_sources = 0;
};
fs_status run_cga(const Graph &g, CgaResult &r);
fs_status build_check_data(const Graph &g, uint32_t flags, ChecksData &cd);
fs_status parse_check_data(const Graph &g, const int32_t *data, uint64_t len, ChecksData &cd);
fs_status build_repair_plan(const Graph &g, const ChecksData &cd, const uint8_t *erased, const uint32_t *want,
                            uint32_t nwant, DecodePlan &pl, RepairStats &rs);
}  // namespace fsb

struct fs_checks {
  fsb::ChecksData cd;
  uint32_t n = 0, K = 0;
};
struct fs_repair_plan {
  fsb::DecodePlan pl;
  fsb::RepairStats rs;
};
