// Internal declarations of libfsb200 (not part of the C ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fsb.h"

namespace fsb {

// ----------------------------------------------------------------- SMEM kernel geometry
// A tile = (stripe, 128-byte slice of every symbol).  Its K intermediate rows are staged
// in shared memory in units of kUnitRows rows (one TMA box of kUnitRows x 128 B each).
constexpr int kSliceBytes = 128;
constexpr int kUnitRows = 32;
constexpr int kUnitBytes = kUnitRows * kSliceBytes;     // 4 KiB
constexpr int kConsumerWarps = 16;
constexpr int kGroupsPerWarp = 4;                        // 8 lanes x 16 B = one 128-B row
constexpr int kGroups = kConsumerWarps * kGroupsPerWarp;
constexpr int kThreads = (kConsumerWarps + 1) * 32;      // + 1 TMA producer warp
constexpr uint16_t kSlotNone = 0xFFFF;
constexpr int kSplitThreshold = 32;                      // rows of degree > this are split
                                                         // over the 4 groups of a warp

// Host-built LT work schedule of the SMEM kernel (identical for every tile).
// Per warp, a run of items.  Item = 16-B header {steps, flags, row0..row3, 0, 0} followed by
// ceil(steps/8) chunks; chunk c = 4 groups x 8 uint16 slots (steps 8c..8c+7 of group g at
// bytes 16*g..16*g+15).  A slot is a tile-relative row (data m -> m, check i -> kpad+i);
// kSlotNone = no edge.  flags bit0 = split item (one row, edges dealt over the 4 groups,
// combined by warp shuffles).
struct SmemSchedule {
  std::vector<uint16_t> words;          // items of all warps, 16-B aligned
  std::vector<uint32_t> warp_begin;     // kConsumerWarps+1 offsets, in 16-B units
  std::vector<uint16_t> pre_slots;      // p * d_p tile-relative data rows
  uint32_t kpad = 0;                    // data rows rounded up to kUnitRows
  uint32_t data_units = 0, check_units = 0, tile_units = 0;
  uint32_t steps_max = 0, steps_total = 0;
};

struct DeviceBufs {
  int device = -1;
  int32_t *pre_row_ptr = nullptr, *pre_col = nullptr, *lt_row_ptr = nullptr, *lt_col = nullptr;
  uint16_t *sched = nullptr;
  uint32_t *warp_begin = nullptr;
  uint16_t *pre_slots = nullptr;
};

struct Graph {
  fs_params prm{};
  std::vector<uint32_t> fin_deg;
  std::vector<double> fin_prob;
  std::vector<int32_t> pre_row_ptr, pre_col, lt_row_ptr, lt_col;
  uint32_t max_degree = 0;
  bool smem_eligible = false;
  SmemSchedule sched;
  DeviceBufs dev;
  int32_t variant = FS_VARIANT_AUTO;
  int sm_count = 0;
  int smem_optin = 0;
  uint32_t smem_bytes = 0;   // dynamic smem of the SMEM kernel
  uint32_t ring_units = 0;   // shared-memory units of the SMEM kernel
};

// fsb_graph.cpp
fs_status validate_params(const fs_params &prm);
fs_status build_cdf(const fs_params &prm, std::vector<uint32_t> &deg, std::vector<double> &cdf);
fs_status generate_csr(Graph &g);
fs_status validate_csr(const Graph &g);
void build_smem_schedule(Graph &g);

// fsb_kernels.cu
fs_status upload_graph(Graph &g);
void free_device(Graph &g);
fs_status launch_encode(const Graph &g, uint32_t S, const uint8_t *data, uint64_t data_stride,
                        uint8_t *checks, uint64_t checks_stride, uint8_t *coded,
                        uint64_t coded_stride, uint32_t row_begin, uint32_t row_end, void *stream,
                        uint32_t *launches);

// fsb_capi.cpp
void set_error(const std::string &msg);

}  // namespace fsb

struct fs_graph {
  fsb::Graph g;
};
