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
constexpr int kSplitThreshold = 32;                      // rows of degree > this are split
                                                         // over the 4 groups of a warp
// Register-resident schedule: each warp keeps its whole per-tile step stream in registers
// (kSchedRegsMax 32-bit words per lane = 16 steps per word) and fetches step e of its lane
// group with one warp shuffle.
constexpr int kStepsPerReg = 16;
constexpr int kSchedRegsMax = 32;
constexpr uint32_t kMaxWarpSteps = kStepsPerReg * kSchedRegsMax;
// 16-bit step values (one per lane group and step):
constexpr uint16_t kIdle = 0x7FFF;        // no edge this step (row shorter than the item)
constexpr uint16_t kStoreFlag = 0x8000;   // store step: 0x8000 | row  (row < 0x4000)
constexpr uint16_t kSplitFlag = 0x4000;   //   split item: 0xC000 | row in all four groups
constexpr uint16_t kStoreNone = 0xBFFF;   //   store step, nothing to store (row 0x3FFF; no split bit)
constexpr uint32_t kMaxSmemRows = 0x3FFF; // n limit of the SMEM variant (rows 0..0x3FFE)
constexpr uint32_t kMaxSmemSlots = 0x7FFE;

// Host-built LT work schedule of the SMEM kernel (identical for every tile).
// Rows of degree > kSplitThreshold are "split" items: their edges are dealt over the 4
// lane groups of a warp and the partial XORs combined with two warp shuffles.  Other rows
// are sorted by degree and packed 4 per item (one per 8-lane group) so the groups of a warp
// run nearly equal edge counts in lockstep.  Items are dealt to warps longest-first onto
// the least-loaded warp (LPT).  Each warp's stream is a sequence of steps; a step holds one
// 16-bit value per group: a tile-relative source row (data m -> m, check i -> kpad+i), kIdle,
// or (after an item's last edge) a store marker.  Stored as 32-bit words: step e, group g
// is the (g&1) half of word 2e + (g>>1) of the warp's stream (see fsb_smem_encode).
struct SmemSchedule {
  std::vector<uint32_t> words;          // kConsumerWarps x (regs*32) words
  std::vector<uint32_t> warp_steps;     // steps per warp (incl. store steps)
  std::vector<uint16_t> pre_slots;      // p * d_p tile-relative data rows
  uint32_t regs = 0;                    // 32-bit schedule registers per lane (16 or 32)
  uint32_t kpad = 0;                    // data rows rounded up to kUnitRows
  uint32_t data_units = 0, check_units = 0, tile_units = 0;
  uint32_t steps_max = 0, steps_total = 0;
};

struct DeviceBufs {
  int device = -1;
  int32_t *pre_row_ptr = nullptr, *pre_col = nullptr, *lt_row_ptr = nullptr, *lt_col = nullptr;
  uint32_t *sched = nullptr;
  uint32_t *warp_steps = nullptr;
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
