// sm_100a kernels of the Founsure encode path (§2.2 steps (1) and (2)).
//
//   precode   C_i = XOR_{m in P(i)} D_m              (a3)
//   LT        Y_j = XOR_{m in N(j)} I_m, I = D ++ C   (a4)
//   stripes   the same graph over every stripe       (a5)
//
// Two variants, bit-identical output (XOR is exact and order-free):
//
// SMEM  (fsb_smem_encode): persistent, one CTA per SM.  A tile = (stripe, 64-byte slice of
//       every symbol).  A TMA warp streams the tile's k data rows (64 rows x 64 B per
//       cp.async.bulk.tensor box) into one of two tile buffers; 3 precode warps compute the p
//       checks from shared memory (written back to smem and HBM); 24 consumer warps compute
//       every coded row as a register XOR of 16-B lanes gathered from shared memory.  Tiles
//       come in pairs (the two 64-B halves of a 128-B column): the first tile's row results
//       are parked in tensor memory, the second tile stores every row as one full 128-B line.
//       HBM sees each source byte once and each output byte once (the ideal one-read-one-write
//       roofline); the gathers hit shared memory only.  Work per warp comes from a host-built,
//       degree-aware schedule (fsb_graph.cpp): light rows are paired by even/odd source counts
//       (bank rule), heavy rows split over two or eight half-groups and recombined by shuffles.
//
// GLOBAL (fsb_precode_global + fsb_lt_band): no staging; every group of 8 lanes XORs one
//       (row, 128-B slice) by 16-B loads from global memory, with the launch rasterised
//       band-major (512-B bands of the symbols) so the band of the source block stays
//       resident in L2 while every row consumes it.  Used for single large stripes
//       (config 5: the 410 MB source exceeds both shared memory and L2) and small calls.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "fsb_internal.h"


namespace fsb {

// --------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Wait for the phase with the given parity.  The suspend-time hint lets the thread sleep in
// hardware until the phase completes instead of polling the barrier word.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "n"(1000000)
        : "memory");
  } while (!done);
}
// Wait with a fixed sleep between probes, for warps that are early and have nothing else to do:
// each probe reads the barrier through the shared-memory pipe, so fast polling (or a suspend that
// wakes on every barrier event in the CTA) steals pipe cycles from the warps still computing.
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity, uint32_t ns) {
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar(uint32_t nconsumer) {
  asm volatile("bar.sync 1, %0;" ::"r"(nconsumer * 32) : "memory");
}
__device__ __forceinline__ void xor_into(uint4 &a, const uint4 &b) {
  a.x ^= b.x;
  a.y ^= b.y;
  a.z ^= b.z;
  a.w ^= b.w;
}
__device__ __forceinline__ void st_stream(uint8_t *p, const uint4 &v) {
  __stcs(reinterpret_cast<uint4 *>(p), v);
}
// 32 contiguous bytes (lo = the first 16): one 256-bit streaming store when the caller's coded
// buffer is 32-B aligned (base and stride; warp-uniform), else two 128-bit ones
__device__ __forceinline__ void st_stream32(uint8_t *p, const uint4 &lo, const uint4 &hi, bool st256) {
  if (st256) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(lo.x), "r"(lo.y),
                 "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
  } else {
    st_stream(p, lo);
    st_stream(p + 16, hi);
  }
}
// 32 B per lane at 8 consecutive 32-bit columns of this warp's lane quarter
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint4 &lo, const uint4 &hi) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(lo.x), "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint4 &lo, uint4 &hi) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
      : "r"(taddr)
      : "memory");
}
// Tensor memory (TMEM): 16 B per lane at 4 consecutive 32-bit columns of this warp's lane quarter.
// tcgen05.ld/st do not use the L1TEX/LSU pipe the gathers saturate (tools/microbench/mb8.cu).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint4 &v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 tmem_ld16(uint32_t taddr) {
  uint4 v;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "r"(taddr)
      : "memory");
  return v;
}

// ============================================================================ SMEM kernel
// Profiling experiments only (FSB_DEBUG=2): per consumer warp, cycles spent waiting for a tile
// (ready/full barriers) and total cycles, summed over CTAs (read with fs_debug_counters).
#ifdef FSB_EXPERIMENTS
// FSB_DEBUG bit 4 (experiment builds, tools/gpu/timeline.py): per-CTA %globaltimer stamps from
// index 64, 16 per CTA (entry, prologue done, first tile ready, mean / last consumer end, last TMA
// issue, %smid, tiles, TMEM allocated, schedule staged, TMA thread past griddepcontrol.wait,
// before / after the prologue barrier)
constexpr uint32_t kDebugCounters = 64 + 16 * 256 + 2 * 128 * 8;
// FSB_DEBUG bit 8: per-tile log of CTAs 0 and gridDim/2 from index 64 + 16*256, 8 per tile (tiles
// < 128): TMA issue done, full seen, ready arrived, consumer start min / max, end min / max
// (min stored as ~t so atomicMax keeps it)
#define FSB_TLOG(stmt) stmt
#define FSB_TL(stmt) stmt
#else
constexpr uint32_t kDebugCounters = 64;
#define FSB_TL(stmt)
#define FSB_TLOG(stmt)
#endif
__device__ unsigned long long g_debug_counters[kDebugCounters];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
struct SmemArgs {
  const uint4 *sched;          // heads ++ conts chunk streams (fsb_internal.h: SmemSchedule)
  const uint32_t *warp_info;   // nc x {items, head_off, cont_off}
  const uint16_t *pre_slots;   // p * d_p tile rows (data, or an earlier check)
  const uint32_t *pre_level_ptr;  // precode levels (nlevels+1 row offsets)
  uint32_t pre_levels;
  uint8_t *checks;
  uint64_t checks_stride;
  uint8_t *coded;
  uint64_t coded_stride;
  uint64_t t;
  uint32_t nslices, ntiles, p, d_p, kpad, zero_even, data_units, tile_units;
  uint32_t slice0;             // first 64-B slice of the column range
  uint32_t sched_chunks, cont_base;
  uint32_t paired;             // 1: tiles come in adjacent-slice pairs, full 128-B line stores
  uint32_t pair_tiles;         // paired: tiles per CTA run as pairs (even); the rest are tail singles
  uint32_t tail_tiles;         // paired: single (unpaired) tiles after the pair rounds, over all CTAs
  uint32_t tmem_cols;          // TMEM columns allocated per CTA in paired mode (power of 2)
  uint32_t debug;              // FSB_DEBUG bits (profiling experiments only; 0 in production)
  uint32_t wait_ns;            // consumer sleep between probes of a tile's `ready` barrier
  uint32_t nc;                 // consumer warps (0..nc-1); warp nc = TMA; warps nc+1.. = precode
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4 &v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Shared address of slot h (0..7) of chunk c: word h/2 holds slots a | b << 21 (fsb_internal.h);
// tile row r lives at sbase + r*64.  h is a compile-time constant after unrolling.  Written in
// PTX so ptxas sees the shift-adds (LEA / LEA.HI) instead of LLVM's canonical shl+and.
__device__ __forceinline__ uint32_t slot_addr(const uint4 &c, int h, uint32_t sbase) {
  const uint32_t w = (h >> 1) == 0 ? c.x : (h >> 1) == 1 ? c.y : (h >> 1) == 2 ? c.z : c.w;
  uint32_t addr;
  if (h & 1) {  // b = w >> 21, bits 11..20 zero: sbase + (w >> 15)
    asm("{\n .reg .b32 t;\n shr.b32 t, %1, 15;\n add.u32 %0, t, %2;\n}" : "=r"(addr) : "r"(w), "r"(sbase));
  } else {      // a = w & 0x7FF: sbase + (a << 6)
    asm("{\n .reg .b32 t;\n and.b32 t, %1, 2047;\n mad.lo.u32 %0, t, 64, %2;\n}" : "=r"(addr) : "r"(w), "r"(sbase));
  }
  return addr;
}

// accA / accB ^= the lane's two 16-B pieces of the tile rows named by slots [H0, H0+N) of chunk
// c: piece at sbase + row*64 and the one at (that ^ 16) -- sbase carries 32*l2 + 16*(g & 1), so the
// lane reads pieces 2*l2 + (g&1) and 2*l2 + 1 - (g&1) (bank rule, fsb_internal.h).  All 2N loads
// are issued before the XOR chains so they overlap.
template <int H0, int N>
__device__ __forceinline__ void gather2(uint4 &accA, uint4 &accB, const uint4 &c, uint32_t sbase) {
  uint4 x[N], y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t a = slot_addr(c, H0 + i, sbase);
    x[i] = lds128(a);
    y[i] = lds128(a ^ 16u);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    xor_into(accA, x[i]);
    xor_into(accB, y[i]);
  }
}

// slots [H0, H0 + n) of chunk c, 1 <= n <= min(4, 8 - H0)
template <int H0>
__device__ __forceinline__ void gather2_n(uint4 &accA, uint4 &accB, const uint4 &c, uint32_t n, uint32_t sbase) {
  switch (n) {
    case 1: gather2<H0, 1>(accA, accB, c, sbase); break;
    case 2: gather2<H0, 2>(accA, accB, c, sbase); break;
    case 3: if (H0 + 3 <= 8) gather2<H0, (H0 + 3 <= 8 ? 3 : 1)>(accA, accB, c, sbase); break;
    default: if (H0 + 4 <= 8) gather2<H0, (H0 + 4 <= 8 ? 4 : 1)>(accA, accB, c, sbase); break;
  }
}

__device__ __forceinline__ void shfl_xor_into(uint4 &a, int o) {
  a.x ^= __shfl_xor_sync(0xffffffffu, a.x, o);
  a.y ^= __shfl_xor_sync(0xffffffffu, a.y, o);
  a.z ^= __shfl_xor_sync(0xffffffffu, a.z, o);
  a.w ^= __shfl_xor_sync(0xffffffffu, a.w, o);
}

// One item (fsb_internal.h): head chunk h, continuation chunks at *cp (shared address, advanced),
// XOR in registers, then the row results leave according to kMode:
// (kMode is warp-uniform and a runtime value: one inlined copy serves all three modes)
//   0 (unpaired): one 64-B store per group (split items: combined over the halves);
//   1 (paired, the pair's first tile): nothing leaves; each lane parks its 32 B in TMEM block `tcol`;
//   2 (paired, second tile = the other 64-B half of the same 128-B lines, read with group g^1's
//     schedule, so group g holds row R_{g^1}): each row leaves as one full 128-B line -- the first
//     tile's half from TMEM (the lane's own row) next to the partner group's second half -- two
//     256-bit stores per lane and item.
// base + row * t in one IMAD.WIDE.U32 (row, t < 2^32)
__device__ __forceinline__ uint8_t *row_addr(uint8_t *base, uint32_t row, uint32_t t) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(row), "r"(t), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<uint8_t *>(r);
}
__device__ __forceinline__ void lt_item(const uint4 &h, uint32_t &cp, uint32_t sbase, uint8_t *out1, uint8_t *out2,
                                        uint32_t t, uint32_t grp, uint32_t tcol, int kMode, bool st256) {
  const uint32_t row = h.x & 0xFFFFu;
  const uint32_t ctrl = h.x >> 16;
  const uint32_t L = ctrl & kMaxItemLen;
  uint4 accA = make_uint4(0, 0, 0, 0), accB = make_uint4(0, 0, 0, 0);
  // the first continuation chunk is requested before the head gathers, so its latency overlaps
  // them instead of following them
  uint4 c = make_uint4(0, 0, 0, 0);
  if (L > kHeadSlots) c = lds128(cp);
  gather2_n<2>(accA, accB, h, L < 4 ? L : 4, sbase);  // head slots 0..3
  if (L > 4) gather2_n<6>(accA, accB, h, L < kHeadSlots ? L - 4 : 2, sbase);  // head slots 4..5
  if (L > kHeadSlots) {
    uint32_t rem = L - kHeadSlots;
    cp += kChunkBytes;
    for (; rem > kChunkSlots; rem -= kChunkSlots) {
      const uint4 nx = lds128(cp);  // next chunk in flight while this one is gathered
      cp += kChunkBytes;
      gather2<0, 4>(accA, accB, c, sbase);
      gather2<4, 4>(accA, accB, c, sbase);
      c = nx;
    }
    gather2_n<0>(accA, accB, c, rem < 4 ? rem : 4, sbase);
    if (rem > 4) gather2_n<4>(accA, accB, c, rem - 4, sbase);
  }
  const bool wsplit = ctrl & kSplitBit;
  // the lane's 32 B in byte order: accA holds piece 2*l2 + (g&1), accB the other
  const bool sg = grp & 1;
  uint4 lo = sg ? accB : accA, hi = sg ? accA : accB;
  if (wsplit) {  // warp-split row: combine the sixteen groups' partial XORs (all lanes get it)
#pragma unroll
    for (int o = 2; o <= 16; o <<= 1) {
      shfl_xor_into(lo, o);
      shfl_xor_into(hi, o);
    }
  } else if (ctrl & kPairSplitBit) {  // pair-split: both halves (groups g, g^2) take the other's part
    uint4 oa, ob;
    oa.x = __shfl_xor_sync(0xffffffffu, lo.x, 4);
    oa.y = __shfl_xor_sync(0xffffffffu, lo.y, 4);
    oa.z = __shfl_xor_sync(0xffffffffu, lo.z, 4);
    oa.w = __shfl_xor_sync(0xffffffffu, lo.w, 4);
    ob.x = __shfl_xor_sync(0xffffffffu, hi.x, 4);
    ob.y = __shfl_xor_sync(0xffffffffu, hi.y, 4);
    ob.z = __shfl_xor_sync(0xffffffffu, hi.z, 4);
    ob.w = __shfl_xor_sync(0xffffffffu, hi.w, 4);
    if (h.y & kPairFlag) {
      xor_into(lo, oa);
      xor_into(hi, ob);
    }
  }
  if (kMode == 0) {
    if (wsplit) {
      if (grp == 0) st_stream32(row_addr(out1, row, t), lo, hi, st256);
    } else if (row != kNoRow) {
      st_stream32(row_addr(out1, row, t), lo, hi, st256);
    }
  } else if (kMode == 1) {
    tmem_st32(tcol, lo, hi);
  } else {
    uint4 plo, phi;
    tmem_ld32(tcol, plo, phi);                                            // own row, slice s
    const uint32_t own = __shfl_xor_sync(0xffffffffu, row, 2);            // R_g (row = R_{g^1})
    const bool odd = grp & 1;
    const uint32_t ra = odd ? row : own, rb = odd ? own : row;            // R_{2q}, R_{2q+1}
    // out1 / out2 = this lane's 32 B in the pair's line at the half it writes of R_{2q} / R_{2q+1}
    // line of R_{2q}: even group its first-tile half (TMEM), odd group the second (computed)
    if (ra != kNoRow && (!wsplit || grp < 2)) st_stream32(row_addr(out1, ra, t), odd ? lo : plo, odd ? hi : phi, st256);
    // line of R_{2q+1}: even group the second-tile half (computed), odd group its first (TMEM)
    if (rb != kNoRow && !wsplit) st_stream32(row_addr(out2, rb, t), odd ? plo : lo, odd ? phi : hi, st256);
  }
}

// Tile i of this CTA: (stripe, slice).  Unpaired: tile blockIdx.x + i*gridDim.x of S x nslices.
// Paired: tiles i < pair_tiles are pairs -- pair blockIdx.x + (i/2)*gridDim.x of S x nslices/2,
// slice 2*(pair % (nslices/2)) plus (i&1), flipped on odd CTAs (half the SMs write their lines
// while the other half park, so the HBM write stream stays even) -- and the pairs that do not
// fill a last round of CTAs run as single unpaired tiles, one per CTA (tail_tiles of them), so no
// CTA does a whole pair more than the mean (config 4 on 8 GPUs: 3.46 pairs per CTA on average
// would otherwise take 4).  (Recomputed with two divisions per tile on purpose: an incremental
// iterator kept ~8 more registers live across the consumers' item loop and made config 4 6%
// slower, 0.597 -> 0.631 ms, profiles/r02/ab_r02o.txt.)
__device__ __forceinline__ bool tile_of(const SmemArgs &a, uint32_t i, uint32_t &stripe, uint32_t &slice) {
  if (a.paired) {
    const uint32_t nsp = a.nslices >> 1;
    uint32_t pair, odd;
    if (i < a.pair_tiles) {
      pair = blockIdx.x + (i >> 1) * gridDim.x;
      if (pair >= (a.ntiles >> 1)) return false;
      odd = (i ^ blockIdx.x) & 1;
    } else {
      const uint32_t q = blockIdx.x + (i - a.pair_tiles) * gridDim.x;  // single tile of the tail
      if (q >= a.tail_tiles) return false;
      pair = (a.pair_tiles >> 1) * gridDim.x + (q >> 1);
      odd = q & 1;
    }
    stripe = pair / nsp;
    slice = a.slice0 + 2 * (pair % nsp) + odd;
    return true;
  }
  const uint32_t tile = blockIdx.x + i * gridDim.x;
  if (tile >= a.ntiles) return false;
  stripe = tile / a.nslices;
  slice = a.slice0 + tile % a.nslices;
  return true;
}

// Persistent encode kernel, one CTA per SM.  Shared memory: two tile buffers (tile_units x 4 KiB
// each), the LT schedule, the precode member rows, then the mbarriers and the TMEM address.
// Warp roles:
//   TMA warp (warp nc; nc = 24 consumer warps unless the graph's precode asks for more precode
//     warps, SmemSchedule::nconsumer): lane 0 streams each tile's data rows in by TMA (box
//     kUnitRows x 64 B);
//   precode warps (the last 28 - 1 - nc): the tile's p checks (PAPER.md:91 step (1)) from shared
//     memory into the buffer's check rows and to HBM, level by level, then `ready`;
//   consumer warps (0..nc-1): every LT row (PAPER.md:91 step (2)) of the tile as a
//     register XOR of 64-B rows gathered from shared memory (lt_item: 64-B stores unpaired,
//     TMEM-parked halves and full 128-B lines paired).
// Buffers alternate (tile i uses buffer i&1), so tile i+1 streams in while tile i computes, and a
// consumer warp that finishes tile i early starts tile i+1 without waiting for the others.
// kSt256: the caller's coded rows are 32-B aligned (base and stride), so every lane's 32 B leave in
// one 256-bit store (else two 128-bit ones; a compile-time choice: a runtime flag tested per store
// cost 2.5% on config 4)
// kTmemHeads (paired launches whose TMEM columns allow it): every item's head chunk -- the lane's
// own group's 16 B and its partner group's -- is copied into tensor memory once per CTA and read
// from there with tcgen05.ld, off the shared-memory port (the continuation chunks stay in shared
// memory).
template <bool kSt256, bool kTmemHeads>
__global__ void __launch_bounds__(kThreads, 1)
    fsb_smem_encode(const __grid_constant__ CUtensorMap tmap, const SmemArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t T = a.tile_units;
  const uint32_t buf_bytes = T * kUnitBytes;
  uint8_t *sched_s = smem + 2 * static_cast<size_t>(buf_bytes);
  uint16_t *pre_s = reinterpret_cast<uint16_t *>(sched_s + static_cast<size_t>(a.sched_chunks) * kChunkBytes);
  const uint32_t pre_n = a.p * a.d_p;
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(pre_s) + ((pre_n * 2 + 15) & ~15u));
  uint64_t *full = bars, *ready = bars + 2, *empty = bars + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6);  // TMEM base address (paired mode)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t smem_base = smem_u32(smem);
  FSB_TL(unsigned long long *tl = g_debug_counters + 64 + 16 * (blockIdx.x & 255);)
  FSB_TLOG(unsigned long long *tlog = (a.debug & 8) && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2)
                                          ? g_debug_counters + 64 + 16 * 256 + (blockIdx.x ? 128 * 8 : 0)
                                          : nullptr;)
  FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) {
    tl[0] = gtime();
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tl[6] = smid;
  })
  if (a.paired && warp == 0) {  // one warp allocates the CTA's TMEM columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    FSB_TL(if ((a.debug & 4) && lane == 0) tl[8] = gtime();)
  }

  const int nc = static_cast<int>(a.nc);
  const uint32_t npw = kConsumerWarps + kPrecodeWarps - a.nc;  // precode warps
  if (warp == nc && lane == 0) {
    // the TMA thread: barriers, then -- once the previous grid in the stream has completed (this
    // prologue may overlap its tail: programmatic dependent launch) -- tile 0's loads, issued
    // while the other threads stage the schedule
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&full[b]), 1);
      mbar_init(smem_u32(&ready[b]), 1);
      mbar_init(smem_u32(&empty[b]), a.nc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    FSB_TL(if (a.debug & 4) tl[10] = gtime();)
    uint32_t stripe, slice;
    if (tile_of(a, 0, stripe, slice)) {  // buffer 0 is free: no wait on `empty`
      if (a.debug & 1) {
        mbar_arrive(smem_u32(&full[0]));
      } else {
        mbar_arrive_expect_tx(smem_u32(&full[0]), a.data_units * kUnitBytes);
        for (uint32_t u = 0; u < a.data_units; ++u)
          tma_load_3d(smem_base + u * kUnitBytes, &tmap, smem_u32(&full[0]), static_cast<int32_t>(slice * kSliceBytes),
                      static_cast<int32_t>(u * kUnitRows), static_cast<int32_t>(stripe));
      }
      FSB_TLOG(if (tlog) tlog[0] = gtime();)
    }
  }
  // the schedule (identical for every tile) and the two zero rows of each buffer
  {  // 4 loads in flight per thread, then their stores (the copy is on every launch's critical path)
    const uint32_t nx = a.sched_chunks * (kChunkBytes / 16);
    for (uint32_t x0 = threadIdx.x; x0 < nx; x0 += 4 * blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t x = x0 + u * blockDim.x;
        if (x < nx) v[u] = __ldg(a.sched + x);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t x = x0 + u * blockDim.x;
        if (x < nx) sts128(smem_u32(sched_s) + x * 16, v[u]);
      }
    }
  }
  FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) tl[9] = gtime();)
  for (uint32_t x = threadIdx.x; x < pre_n; x += blockDim.x) pre_s[x] = __ldg(&a.pre_slots[x]);
  if (threadIdx.x < 2 * 2 * (kSliceBytes / 16)) {  // 2 buffers x 2 rows x 4 lanes
    const uint32_t b = threadIdx.x >> 3, r = (threadIdx.x >> 2) & 1, l4 = threadIdx.x & 3;
    sts128(smem_base + b * buf_bytes + (a.zero_even + r) * kSliceBytes + l4 * 16, make_uint4(0, 0, 0, 0));
  }
  FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) tl[12] = gtime();)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) tl[13] = gtime();)
  // every thread past this point reads or writes user buffers after the previous grid is done;
  // the next launch may then start its prologue on SMs as they free up
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) tl[1] = gtime();)

  if (warp == nc) {
    // ---------------------------------------------------------------- TMA warp (one lane)
    if (lane == 0) {
      uint32_t stripe, slice;
      for (uint32_t i = 1; tile_of(a, i, stripe, slice); ++i) {  // tile 0: issued above
        const uint32_t b = i & 1, ph = (i >> 1) & 1;
        const uint32_t buf = smem_base + b * buf_bytes;
        const long long tw0 = (a.debug & 2) ? clock64() : 0;
        mbar_wait(smem_u32(&empty[b]), ph ^ 1);  // consumers released tile i-2
        if (a.debug & 2) atomicAdd(&g_debug_counters[60], static_cast<unsigned long long>(clock64() - tw0));
        if (a.debug & 1) {  // experiment: no TMA (consumers gather stale rows)
          mbar_arrive(smem_u32(&full[b]));
        } else {
          mbar_arrive_expect_tx(smem_u32(&full[b]), a.data_units * kUnitBytes);
        }
        for (uint32_t u = 0; u < a.data_units && !(a.debug & 1); ++u)
          tma_load_3d(buf + u * kUnitBytes, &tmap, smem_u32(&full[b]), static_cast<int32_t>(slice * kSliceBytes),
                      static_cast<int32_t>(u * kUnitRows), static_cast<int32_t>(stripe));
        FSB_TLOG(if (tlog && i < 128) tlog[i * 8 + 0] = gtime();)
      }
      FSB_TL(if (a.debug & 4) tl[5] = gtime();)
    }
    return;
  }
  if (warp > nc) {
    // ----------------------------------------------------------- precode warps (a3, Check #1)
    // After a tile's rows land: its p checks (PAPER.md:91 step (1)) from shared memory into the
    // buffer's check rows and to HBM, level by level (Alg 2 checks read earlier checks), then
    // `ready`.  Separate from the TMA warp so the next tile's loads never wait for this work.
    const uint32_t pw = warp - nc - 1;                              // precode warp 0..npw-1
    const uint32_t half_id = pw * kHalvesPerWarp + (lane >> 2), lane4 = lane & 3;
    uint32_t stripe, slice;
    const long long pt0 = (a.debug & 2) ? clock64() : 0;
    for (uint32_t i = 0; tile_of(a, i, stripe, slice); ++i) {
      const uint32_t b = i & 1, ph = (i >> 1) & 1;
      const uint32_t buf = smem_base + b * buf_bytes;
      const long long tw0 = (a.debug & 2) ? clock64() : 0;
      mbar_wait(smem_u32(&full[b]), ph);
      if ((a.debug & 2) && lane == 0)
        atomicAdd(&g_debug_counters[48 + 2 * pw], static_cast<unsigned long long>(clock64() - tw0));
      FSB_TLOG(if (tlog && i < 128 && pw == 0 && lane == 0) tlog[i * 8 + 1] = gtime();)
      // precode, level by level (a check may read checks of earlier levels, Alg 2): check c of
      // a level by half-group (c - level start) % 8, 16 B per lane
      const uint32_t lb = buf + lane4 * 16;
      const uint64_t col_off = static_cast<uint64_t>(slice) * kSliceBytes + lane4 * 16;
      for (uint32_t L = 0; L < a.pre_levels; ++L) {
        const uint32_t c0 = __ldg(&a.pre_level_ptr[L]), c1 = __ldg(&a.pre_level_ptr[L + 1]);
        for (uint32_t c = c0 + half_id; c < c1; c += kHalvesPerWarp * npw) {
          uint4 acc = make_uint4(0, 0, 0, 0);
          const uint16_t *ps = pre_s + c * a.d_p;  // member rows, staged in shared memory
          uint32_t e = 0;
          for (; e + 8 <= a.d_p; e += 8) {  // 8 slot loads, then 8 gathers, in flight together
            uint32_t r[8];
            uint4 x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = ps[e + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = lds128(lb + r[u] * kSliceBytes);
#pragma unroll
            for (int u = 0; u < 8; ++u) xor_into(acc, x[u]);
          }
          for (; e < a.d_p; ++e) xor_into(acc, lds128(lb + ps[e] * kSliceBytes));
          sts128(lb + (a.kpad + c) * kSliceBytes, acc);
          st_stream(a.checks + stripe * a.checks_stride + c * a.t + col_off, acc);
        }
        // this level's check rows before the next level reads them (all precode warps)
        asm volatile("bar.sync 2, %0;" ::"r"(npw * 32) : "memory");
      }
      FSB_TLOG(if (tlog && i < 128 && pw == 0 && lane == 0) tlog[i * 8 + 2] = gtime();)
      if (pw == 0 && lane == 0) mbar_arrive(smem_u32(&ready[b]));  // release: data + checks visible
    }
    if ((a.debug & 2) && lane == 0)
      atomicAdd(&g_debug_counters[49 + 2 * pw], static_cast<unsigned long long>(clock64() - pt0));
    return;
  }

  // ------------------------------------------------------------------- consumer warps
  const uint32_t grp = lane >> 1, l2 = lane & 1;  // group (2 lanes, 32 B each, of a 64-B row slice)
  const uint32_t nitems = __ldg(&a.warp_info[warp * 3 + 0]);
  const uint32_t head_b = smem_u32(sched_s) + __ldg(&a.warp_info[warp * 3 + 1]) * kChunkBytes;
  const uint32_t cont_b = smem_u32(sched_s) + (a.cont_base + __ldg(&a.warp_info[warp * 3 + 2])) * kChunkBytes;
  // TMEM: this warp's lane quarter (warp % 4) and its column block after the earlier warps of the
  // same quarter: 8 columns (32 B per lane) per item for the parked results, then (kTmemHeads) 8
  // per item for the head chunks (own group's 16 B, partner group's 16 B)
  constexpr uint32_t kColsPerItem = kTmemHeads ? 16 : 8;
  uint32_t tcol0 = 0, hcol0 = 0;
  if (a.paired) {
    uint32_t col = 0;
    for (int w = warp & 3; w < warp; w += 4) col += kColsPerItem * __ldg(&a.warp_info[w * 3 + 0]);
    tcol0 = *tmem_slot + ((32u * (warp & 3)) << 16) + col;
    hcol0 = tcol0 + 8 * nitems;
  }
  if (kTmemHeads) {
    for (uint32_t it = 0; it < nitems; ++it) {
      tmem_st16(hcol0 + 8 * it, lds128(head_b + it * kChunkBytes + grp * 16));
      tmem_st16(hcol0 + 8 * it + 4, lds128(head_b + it * kChunkBytes + (grp ^ 1) * 16));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  const long long t_start = (a.debug & 2) ? clock64() : 0;
  uint32_t stripe, slice;
  for (uint32_t i = 0; tile_of(a, i, stripe, slice); ++i) {
    const uint32_t b = i & 1, ph = (i >> 1) & 1;
    const int mode = (a.paired && i < a.pair_tiles) ? 1 + (i & 1) : 0;
    const uint32_t first = (blockIdx.x & 1) ? kSliceBytes : 0;  // line offset of the pair's first tile
    // odd tiles of a pair read the partner group's schedule (its rows, their slice s+1)
    const uint32_t hsel = (mode == 2 ? grp ^ 1 : grp) * 16;
    // this lane's first piece of tile row 0 (32 B per lane; pieces ordered by the bank rule)
    const uint32_t sbase = smem_base + b * buf_bytes + l2 * 32 + (grp & 1) * 16;
    uint32_t hp = head_b + hsel, cp = cont_b + hsel;
    uint4 h0 = make_uint4(0, 0, 0, 0);
    if (!kTmemHeads) h0 = lds128(hp);
    long long t_wait0 = 0;
    if (a.debug & 2) t_wait0 = clock64();
    if (a.wait_ns) mbar_wait_backoff(smem_u32(&ready[b]), ph, a.wait_ns);
    else mbar_wait(smem_u32(&ready[b]), ph);  // FSB_WAIT_NS=0: hardware-suspended try_wait
    mbar_wait(smem_u32(&full[b]), ph);
    if ((a.debug & 2) && lane == 0) atomicAdd(&g_debug_counters[warp * 2], static_cast<unsigned long long>(clock64() - t_wait0));
    FSB_TL(if ((a.debug & 4) && i == 0 && threadIdx.x == 0) tl[2] = gtime();)
    FSB_TL(if ((a.debug & 4) && threadIdx.x == 0) tl[7] = i + 1;)
    FSB_TLOG(if (tlog && i < 128 && lane == 0) {
      const unsigned long long tn = gtime();
      atomicMax(&tlog[i * 8 + 3], ~tn);
      atomicMax(&tlog[i * 8 + 4], tn);
    })
    // unpaired: this slice's 64 B; paired: the pair's 128-B line (slice s = the even one), at the
    // half this lane writes of R_{2q} (out1) and of R_{2q+1} (out2) -- `first` = byte offset in the
    // line of the pair's first tile
    uint8_t *out1 = a.coded + stripe * a.coded_stride +
                    static_cast<uint64_t>(mode ? (slice & ~1u) : slice) * kSliceBytes + l2 * 32;
    uint8_t *out2 = out1;
    if (mode) {
      const bool hi = grp & 1;
      out1 += hi ? kSliceBytes - first : first;
      out2 += hi ? first : kSliceBytes - first;
    }
    const uint32_t t32 = static_cast<uint32_t>(a.t);
    if (kTmemHeads) {
      const uint32_t hc = hcol0 + (mode == 2 ? 4 : 0);
      for (uint32_t it = 0; it < nitems; ++it)
        lt_item(tmem_ld16(hc + 8 * it), cp, sbase, out1, out2, t32, grp, tcol0 + 8 * it, mode, kSt256);
    } else {
      // items, with the next head chunk in flight (2-way unrolled so no register moves)
      for (uint32_t it = 0; it < nitems; it += 2) {
        const uint4 h1 = lds128(hp + kChunkBytes);
        lt_item(h0, cp, sbase, out1, out2, t32, grp, tcol0 + 8 * it, mode, kSt256);
        if (it + 1 >= nitems) break;
        h0 = lds128(hp + 2 * kChunkBytes);
        hp += 2 * kChunkBytes;
        lt_item(h1, cp, sbase, out1, out2, t32, grp, tcol0 + 8 * (it + 1), mode, kSt256);
      }
    }
    if (mode == 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // parked before reuse
    __syncwarp();
    FSB_TLOG(if (tlog && i < 128 && lane == 0) {
      const unsigned long long tn = gtime();
      atomicMax(&tlog[i * 8 + 5], ~tn);
      atomicMax(&tlog[i * 8 + 6], tn);
    })
    if (lane == 0) mbar_arrive(smem_u32(&empty[b]));
  }
  if ((a.debug & 2) && lane == 0) atomicAdd(&g_debug_counters[warp * 2 + 1], static_cast<unsigned long long>(clock64() - t_start));
  FSB_TL(if ((a.debug & 4) && lane == 0) {
    const unsigned long long te = gtime();
    atomicAdd(&tl[3], te / a.nc);
    atomicMax(&tl[4], te);
  })
  if (a.paired) {  // all consumer warps are done with TMEM; warp 0 frees it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    consumer_bar(a.nc);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(a.tmem_cols)
                   : "memory");
  }
}

// ========================================================================= GLOBAL kernels
constexpr int kGlobalThreads = 256;
constexpr int kGroupsPerBlock = kGlobalThreads / 8;
constexpr uint32_t kGSliceBytes = 128;  // one 8-lane group = 8 x 16 B

// Checks [c0, c0 + nc) of one precode level: one 8-lane group per (stripe, check, 128-B slice).
// A member m >= k is a check of an earlier level (Alg 2), read from the checks buffer.
__global__ void __launch_bounds__(kGlobalThreads)
    fsb_precode_global(uint32_t S, uint32_t c0, uint32_t nc, uint32_t k, uint32_t d_p, uint64_t t, uint64_t col0,
                       uint64_t col1, uint32_t nslices, const int32_t *__restrict__ pre_col, const uint8_t *__restrict__ data,
                       uint64_t data_stride, uint8_t *checks, uint64_t checks_stride) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // an earlier precode level (PDL)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t item = static_cast<uint64_t>(blockIdx.x) * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint32_t lane8 = threadIdx.x & 7;
  const uint64_t total = static_cast<uint64_t>(S) * nc * nslices;
  if (item >= total) return;
  const uint32_t slice = item % nslices;
  const uint64_t r = item / nslices;
  const uint32_t c = c0 + static_cast<uint32_t>(r % nc);
  const uint32_t s = static_cast<uint32_t>(r / nc);
  const uint64_t byte = col0 + static_cast<uint64_t>(slice) * kGSliceBytes + lane8 * 16;
  if (byte >= col1) return;
  const uint8_t *src = data + s * data_stride + byte;
  const uint8_t *csrc = checks + s * checks_stride + byte;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint32_t e = 0; e < d_p; ++e) {
    const uint32_t m = static_cast<uint32_t>(__ldg(&pre_col[c * d_p + e]));
    const uint4 *p = reinterpret_cast<const uint4 *>(m < k ? src + static_cast<uint64_t>(m) * t
                                                           : csrc + static_cast<uint64_t>(m - k) * t);
    xor_into(acc, m < k ? __ldg(p) : *p);  // checks were written by an earlier launch
  }
  *reinterpret_cast<uint4 *>(checks + s * checks_stride + static_cast<uint64_t>(c) * t + byte) = acc;
}

// LT rows of one (stripe, 512-B band) per warp and chunk of kBandRows consecutive coded rows.
// Lane l owns bytes [band*512 + 16l, +16) of every row.  The chunk's CSR column indices are read
// 32 at a time with one coalesced load and broadcast by shuffles, so the 512-B source gathers
// (16 B per lane, 4 full lines per warp load) are independent of any other global load and go out
// kBandBatch at a time.  Warps are ordered band-major (the unit index runs over chunks fastest),
// so all SMs sweep the same band of the source block, which stays resident in L2 (config 5: a
// 512-B band of all 50,500 rows is 25.9 MB) while every coded row consumes it: HBM reads the
// source about once, the gathers hit L2.
constexpr uint32_t kBandBytes = 512;
constexpr uint32_t kBandRowsMax = 8;   // coded rows per warp (fewer when the call is small)
constexpr uint32_t kQBandBytes = 128;  // band of the four-group long-row level kernel

template <uint32_t kBandBatch, int kMinBlocks, bool kLazyWait>
__global__ void __launch_bounds__(kGlobalThreads, kMinBlocks)
    fsb_lt_band(uint32_t S, uint32_t k, uint32_t t, uint32_t col0, uint32_t col1, uint32_t nbands, uint32_t row_begin,
                uint32_t nrows, uint32_t band_rows, const int32_t *__restrict__ row_ptr, const uint32_t *__restrict__ colf,
                const uint8_t *__restrict__ data, uint64_t data_stride, const uint8_t *__restrict__ checks,
                uint64_t checks_stride, uint8_t *__restrict__ coded, uint64_t coded_stride) {
  // launched programmatically after the precode kernel (PDL): the CTAs are scheduled while it
  // drains.  kLazyWait (few-wave calls): a warp waits for the precode grid only before its first
  // batch that reads a check row, so rows of data sources alone proceed while the checks are
  // computed (config 3: 32.6 -> 30.2 us); otherwise every warp waits at entry (config 5, 13
  // waves: the early warps' gathers slowed the precode, 0.281 -> 0.288 ms).  The source loads
  // are asm volatile, like the wait, so the compiler cannot move them above it (an invariant
  // __ldg could be hoisted -- a first version read checks before they existed that way).
  if (!kLazyWait) asm volatile("griddepcontrol.wait;" ::: "memory");
  bool waited = !kLazyWait;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nchunks = (nrows + band_rows - 1) / band_rows;
  uint64_t unit = static_cast<uint64_t>(blockIdx.x) * (kGlobalThreads / 32) + (threadIdx.x >> 5);
  const uint32_t chunk = static_cast<uint32_t>(unit % nchunks);
  unit /= nchunks;
  const uint32_t band = static_cast<uint32_t>(unit % nbands);
  const uint64_t s = unit / nbands;
  if (s >= S) return;
  const uint32_t byte_raw = col0 + band * kBandBytes + lane * 16;  // bands cover columns [col0, col1)
  const bool active = byte_raw < col1;                // ragged last band
  const uint32_t byte = active ? byte_raw : col0;     // inactive lanes load a valid address
  // source row m lives at (m < k ? dbase : cbase) + m*t  (checks: row k+i = check i)
  const uint8_t *dbase = data + s * data_stride + byte;
  const uint8_t *cbase = checks + s * checks_stride + byte - static_cast<uint64_t>(k) * t;
  const uint32_t r0 = chunk * band_rows;              // first row of the chunk (relative)
  const uint32_t rows = min(band_rows, nrows - r0);
  const int32_t base = __ldg(&row_ptr[row_begin + r0]);
  const int32_t end = __ldg(&row_ptr[row_begin + r0 + rows]);
  uint8_t *out = coded + s * coded_stride + static_cast<uint64_t>(r0) * t + byte_raw;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int32_t e0 = base; e0 < end; e0 += 32) {
    // 32 marked column indices (bit 31 = last edge of its row) per coalesced load; positions
    // past `end` read row 0 and are never XORed
    const uint32_t cv = e0 + static_cast<int32_t>(lane) < end ? __ldg(&colf[e0 + lane]) : 0u;
    const int32_t nb = min(32, end - e0);
    for (int32_t kk = 0; kk < nb; kk += kBandBatch) {
      uint4 v[kBandBatch];
      uint32_t mr[kBandBatch];
      bool chk = false;
#pragma unroll
      for (uint32_t u = 0; u < kBandBatch; ++u) {
        mr[u] = __shfl_sync(0xffffffffu, cv, kk + u);
        chk |= (mr[u] & 0x7FFFFFFFu) >= k;  // warp-uniform
      }
      if (chk && !waited) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
      }
#pragma unroll
      for (uint32_t u = 0; u < kBandBatch; ++u) {
        uint32_t m = mr[u] & 0x7FFFFFFFu;
#if defined(FSB_EXPERIMENTS) && defined(FSB_BAND_L2ONLY)
        m &= 1023u;  // experiment: every gather L2-resident (wrong bytes by design)
#endif
        const uint8_t *b0 = m < k ? dbase : cbase;
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(b0 + static_cast<uint64_t>(m) * t));
      }
      const int32_t lim = min(static_cast<int32_t>(kBandBatch), nb - kk);
#pragma unroll
      for (int32_t u = 0; u < static_cast<int32_t>(kBandBatch); ++u) {
        if (u >= lim) break;
        xor_into(acc, v[u]);
        if (mr[u] >> 31) {  // warp-uniform: the row is complete
          if (active) st_stream(out, acc);
          acc = make_uint4(0, 0, 0, 0);
          out += t;
        }
      }
    }
  }
}

// The source address of marked edge f: data row m < k or check row m - k (cbase = checks - k*t).
__device__ __forceinline__ const uint8_t *src_addr(uint32_t f, uint32_t k, uint32_t t, const uint8_t *dbase,
                                                   const uint8_t *cbase) {
  uint32_t m = f & 0x7FFFFFFFu;
#if defined(FSB_EXPERIMENTS) && defined(FSB_BAND_L2ONLY)
  m &= 1023u;  // experiment: every gather L2-resident (wrong bytes by design)
#endif
  return (m < k ? dbase : cbase) + static_cast<uint64_t>(m) * t;
}
__device__ __forceinline__ uint4 ldg16(const uint8_t *p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// fsb_lt_band4: the band kernel for many-wave calls (config 5).  Same units, band-major order and
// marked CSR as fsb_lt_band; kB gathers per batch.  A chunk's edge count modulo kB is taken first
// as one predicated partial batch, so every later batch issues kB unpredicated gathers, and row
// ends inside a batch are found with one warp vote (the flags are warp-uniform).  Stores are
// plain write-back st.global: in an L2 gather stream with one 512-B store per 8 gathers, .cs
// stores cost ~6% of the gather rate (tools/microbench/mb11.cu, profiles/r02).
template <int kB>
__device__ __forceinline__ void band_batch(uint4 &acc, const uint32_t (&f)[kB], const uint4 (&v)[kB], uint8_t *&out,
                                           uint32_t t, bool active, uint32_t lane) {
  uint32_t sel = 0;
#pragma unroll
  for (int u = 0; u < kB; ++u) sel = lane == static_cast<uint32_t>(u) ? f[u] : sel;
  const uint32_t ends = __ballot_sync(0xffffffffu, lane < static_cast<uint32_t>(kB) && static_cast<int32_t>(sel) < 0);
  if (ends == 0u) {
#pragma unroll
    for (int u = 0; u + 1 < kB; u += 2) {
      acc.x ^= v[u].x ^ v[u + 1].x;
      acc.y ^= v[u].y ^ v[u + 1].y;
      acc.z ^= v[u].z ^ v[u + 1].z;
      acc.w ^= v[u].w ^ v[u + 1].w;
    }
    if (kB & 1) xor_into(acc, v[kB - 1]);
  } else {
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      xor_into(acc, v[u]);
      if (ends & (1u << u)) {
        if (active) *reinterpret_cast<uint4 *>(out) = acc;
        out += t;
        acc = make_uint4(0, 0, 0, 0);
      }
    }
  }
}

constexpr int kBand4Threads = 64;  // 2-warp blocks: a block slot frees as soon as its 2 warps finish
template <int kB, int kMinBlocks, int kBT = kGlobalThreads>
__global__ void __launch_bounds__(kBT, kMinBlocks)
    fsb_lt_band4(uint32_t S, uint32_t k, uint32_t t, uint32_t col0, uint32_t col1, uint32_t nbands, uint32_t row_begin,
                 uint32_t nrows, uint32_t band_rows, const int32_t *__restrict__ row_ptr,
                 const uint32_t *__restrict__ colf, const uint8_t *__restrict__ data, uint64_t data_stride,
                 const uint8_t *__restrict__ checks, uint64_t checks_stride, uint8_t *__restrict__ coded,
                 uint64_t coded_stride) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the precode launch (PDL)
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nchunks = (nrows + band_rows - 1) / band_rows;
  const uint32_t unit = blockIdx.x * (kBT / 32) + (threadIdx.x >> 5);  // < 2^31 (host check)
  const uint32_t chunk = unit % nchunks;
  const uint32_t rest = unit / nchunks;
  const uint32_t band = rest % nbands;
  const uint32_t s = rest / nbands;
  if (s >= S) return;
  const uint32_t byte_raw = col0 + band * kBandBytes + lane * 16;
  const bool active = byte_raw < col1;
  const uint32_t byte = active ? byte_raw : col0;
  const uint8_t *dbase = data + s * data_stride + byte;
  const uint8_t *cbase = checks + s * checks_stride + byte - static_cast<uint64_t>(k) * t;
  const uint32_t r0 = chunk * band_rows;
  const uint32_t rows = min(band_rows, nrows - r0);
  const int32_t base = __ldg(&row_ptr[row_begin + r0]);
  const int32_t end = __ldg(&row_ptr[row_begin + r0 + rows]);
  uint8_t *out = coded + s * coded_stride + static_cast<uint64_t>(r0) * t + byte_raw;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int32_t head = (end - base) % kB;  // the partial batch, first
  int32_t e0 = base;
  uint32_t cv = static_cast<int32_t>(lane) < end - base ? __ldg(&colf[base + lane]) : 0u;
  int32_t kk = 0;
  if (head) {
    uint32_t f[kB];
    uint4 v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      f[u] = __shfl_sync(0xffffffffu, cv, u);
      if (u >= head) f[u] = 0;
      v[u] = make_uint4(0, 0, 0, 0);
      if (u < head) v[u] = ldg16(src_addr(f[u], k, t, dbase, cbase));
    }
    band_batch<kB>(acc, f, v, out, t, active, lane);
    kk = head;
  }
  while (e0 < end) {  // windows of up to 32 indices; after the head every batch is full
    const int32_t nb = min(32, end - e0);
    for (; kk + kB <= nb; kk += kB) {
      uint32_t f[kB];
      uint4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        f[u] = __shfl_sync(0xffffffffu, cv, (kk + u) & 31);
        v[u] = ldg16(src_addr(f[u], k, t, dbase, cbase));
      }
      band_batch<kB>(acc, f, v, out, t, active, lane);
    }
    e0 += kk;
    kk = 0;
    cv = static_cast<int32_t>(lane) < end - e0 ? __ldg(&colf[e0 + lane]) : 0u;
  }
}

// fsb_lt_win: the band kernel over fixed-size edge windows (round 2).  The host packs the LT rows
// into windows of at most 32 x kWR marked edges and a few whole rows (fsb_internal.h: LtWindows);
// a warp takes one (stripe, 512-B band, window), so the window's edges sit at
// went[w * 32 * kWR] and its first row in whdr[w]: both loads depend only on the warp's unit
// index and go out together, where fsb_lt_band4 first reads row_ptr and only then the edge
// indices (two dependent L2 round trips before the first gather).  Each window's edge count is
// padded to a multiple of 4 with skip entries at its start (bit 30), so every batch of 4 sits
// aligned inside one 32-edge register and only the first batch is predicated.  A window may start
// before row_begin or end after row_end (row-range calls, kRange): rows outside the range are
// computed but not stored.
#ifndef FSB_WIN_POLICY
#define FSB_WIN_POLICY 1  // 1 = source loads with an L2 evict_last policy (default; A/B: config 3 21.6 -> 19.5 us, config 5 unchanged); 2 = row stores evict_first (experiments)
#endif
__device__ __forceinline__ uint4 ldg16_pol(const uint8_t *p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg16_pol(uint8_t *p, const uint4 &v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

template <int kB, bool kRange>
__device__ __forceinline__ void win_batch(uint4 &acc, const uint32_t (&f)[kB], const uint4 (&v)[kB], uint8_t *&out,
                                          uint32_t t, bool active, uint32_t lane, uint32_t &row, uint32_t rb,
                                          uint32_t re) {
  uint32_t sel = 0;
#pragma unroll
  for (int u = 0; u < kB; ++u) sel = lane == static_cast<uint32_t>(u) ? f[u] : sel;
  const uint32_t ends = __ballot_sync(0xffffffffu, lane < static_cast<uint32_t>(kB) && static_cast<int32_t>(sel) < 0);
  if (ends == 0u) {
#pragma unroll
    for (int u = 0; u + 1 < kB; u += 2) {
      acc.x ^= v[u].x ^ v[u + 1].x;
      acc.y ^= v[u].y ^ v[u + 1].y;
      acc.z ^= v[u].z ^ v[u + 1].z;
      acc.w ^= v[u].w ^ v[u + 1].w;
    }
    if (kB & 1) xor_into(acc, v[kB - 1]);
  } else {
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      xor_into(acc, v[u]);
      if (ends & (1u << u)) {
        if (active && (!kRange || (row >= rb && row < re))) {
#if FSB_WIN_POLICY & 2
          stg16_pol(out, acc, policy_evict_first());
#else
          *reinterpret_cast<uint4 *>(out) = acc;
#endif
        }
        out += t;
        if (kRange) ++row;
        acc = make_uint4(0, 0, 0, 0);
      }
    }
  }
}

template <int kWR, int kMinBlocks, int kBT, bool kRange>
__global__ void __launch_bounds__(kBT, kMinBlocks)
    fsb_lt_win(uint32_t S, uint32_t k, uint32_t t, uint32_t col0, uint32_t col1, uint32_t nbands, uint32_t w0,
               uint32_t nwin, uint32_t row_begin, uint32_t row_end, const uint2 *__restrict__ whdr,
               const uint32_t *__restrict__ went, const uint8_t *__restrict__ data, uint64_t data_stride,
               const uint8_t *__restrict__ checks, uint64_t checks_stride, uint8_t *__restrict__ coded,
               uint64_t coded_stride) {
  constexpr int kB = 4;  // gathers per batch; 8 batches per 32-edge register
#if FSB_WIN_POLICY & 1
  const uint64_t lpol = policy_evict_last();
#define WIN_LDG(p) ldg16_pol((p), lpol)
#else
#define WIN_LDG(p) ldg16(p)
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the precode launch (PDL)
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t unit = blockIdx.x * (kBT / 32) + (threadIdx.x >> 5);  // < 2^31 (host check)
  const uint32_t w = w0 + unit % nwin;
  const uint32_t rest = unit / nwin;
  const uint32_t band = rest % nbands;
  const uint32_t s = rest / nbands;
  if (s >= S) return;
  // the window: header and all its edge slots in one round trip
  const uint32_t *we = went + static_cast<size_t>(w) * (32 * kWR);
  const uint2 h = __ldg(&whdr[w]);
  uint32_t cv[kWR];
#pragma unroll
  for (int r = 0; r < kWR; ++r) cv[r] = __ldg(&we[32 * r + lane]);
  const uint32_t byte_raw = col0 + band * kBandBytes + lane * 16;
  const bool active = byte_raw < col1;
  const uint32_t byte = active ? byte_raw : col0;
  const uint8_t *dbase = data + s * data_stride + byte;
  const uint8_t *cbase = checks + s * checks_stride + byte - static_cast<uint64_t>(k) * t;
  uint32_t row = h.x;
  const uint32_t nb = h.y;  // batches of 4 (>= 1)
  uint8_t *out = coded + s * coded_stride + (static_cast<int64_t>(row) - static_cast<int64_t>(row_begin)) * t + byte_raw;
  uint4 acc = make_uint4(0, 0, 0, 0);
  {  // batch 0: its leading skip entries (bit 30) load nothing
    uint32_t f[kB];
    uint4 v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      f[u] = __shfl_sync(0xffffffffu, cv[0], u);
      v[u] = make_uint4(0, 0, 0, 0);
      if (!(f[u] & kWinSkip)) v[u] = WIN_LDG(src_addr(f[u], k, t, dbase, cbase));
    }
    win_batch<kB, kRange>(acc, f, v, out, t, active, lane, row, row_begin, row_end);
  }
#pragma unroll
  for (int r = 0; r < kWR; ++r) {  // batches 8r .. 8r+7 live in register r
    for (uint32_t b = (r == 0 ? 1 : 0); b < 8 && 8 * r + b < nb; ++b) {
      uint32_t f[kB];
      uint4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        f[u] = __shfl_sync(0xffffffffu, cv[r], b * kB + u);
        v[u] = WIN_LDG(src_addr(f[u], k, t, dbase, cbase));
      }
      win_batch<kB, kRange>(acc, f, v, out, t, active, lane, row, row_begin, row_end);
    }
  }
}

// ====================================================================== decoder (NEXT-1)
// One DPG level (fsb_decode.cpp): row r recovers intermediate symbol target[r] of every stripe as
// the XOR of its sources (intermediate rows recovered at earlier levels, or a received coded
// row).  Same layout and schedule as fsb_lt_band: one warp per (stripe, 512-B band, chunk of
// rows), source indices 32 per coalesced load, bit 31 = a row's last source.
template <uint32_t kBatch, int kMinBlocks>
__global__ void __launch_bounds__(kGlobalThreads, kMinBlocks)
    fsb_dpg_level(uint32_t S, uint32_t t, uint32_t nbands, uint32_t row0, uint32_t nrows, uint32_t band_rows,
                  const int32_t *__restrict__ target, const int32_t *__restrict__ src_ptr,
                  const uint32_t *__restrict__ src, uint8_t *coded, uint64_t coded_stride,
                  uint8_t *inter, uint64_t inter_stride, uint8_t *work, uint64_t work_stride, uint32_t rev) {
  // programmatic dependent launch: this level's CTAs may be scheduled while the previous level
  // drains; they wait here until it has completed and its writes are visible, and let the next
  // level be scheduled as soon as every CTA of this one has started
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nchunks = (nrows + band_rows - 1) / band_rows;
  const uint64_t total = static_cast<uint64_t>(S) * nbands * nchunks;
  uint64_t unit = static_cast<uint64_t>(blockIdx.x) * (kGlobalThreads / 32) + (threadIdx.x >> 5);
  if (unit >= total) return;
  // serpentine: odd levels sweep (stripe, band) backwards, so a level starts on the bands the
  // previous one touched last (still in L2)
  if (rev) unit = total - 1 - unit;
  const uint32_t chunk = static_cast<uint32_t>(unit % nchunks);
  unit /= nchunks;
  const uint32_t band = static_cast<uint32_t>(unit % nbands);
  const uint64_t s = unit / nbands;
  const uint32_t byte_raw = band * kBandBytes + lane * 16;
  const bool active = byte_raw < t;
  const uint32_t byte = active ? byte_raw : 0;
  const uint8_t *ibase = inter + s * inter_stride + byte;  // read: rows of earlier levels
  const uint8_t *cbase = coded + s * coded_stride + byte;
  const uint8_t *wbase = work + s * work_stride + byte;   // read: workspace rows (m | kSrcWork)
  uint8_t *obase = inter + s * inter_stride + byte_raw;  // target m: intermediate row m
  uint8_t *cobase = coded + s * coded_stride + byte_raw; // target m | kSrcCoded: coded row m (repair)
  uint8_t *wobase = work + s * work_stride + byte_raw;   // target m | kSrcWork: workspace row m
  const uint32_t r0 = row0 + chunk * band_rows;
  const uint32_t rows = min(band_rows, row0 + nrows - r0);
  const int32_t tg = lane < rows ? __ldg(&target[r0 + lane]) : 0;
  const int32_t base = __ldg(&src_ptr[r0]);
  const int32_t end = __ldg(&src_ptr[r0 + rows]);
  uint32_t cur = 0;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int32_t e0 = base; e0 < end; e0 += 32) {
    // past-the-end lanes name coded row 0 (always a valid address; d_inter may be NULL in repair)
    const uint32_t cv = e0 + static_cast<int32_t>(lane) < end ? __ldg(&src[e0 + lane]) : kSrcCoded;
    const int32_t nb = min(32, end - e0);
    for (int32_t kk = 0; kk < nb; kk += kBatch) {
      uint4 v[kBatch];
      uint32_t fl[kBatch];
#pragma unroll
      for (uint32_t u = 0; u < kBatch; ++u) {
        fl[u] = __shfl_sync(0xffffffffu, cv, kk + u);
        const uint32_t m = fl[u] & kSrcIndex;
        const uint8_t *b0 = (fl[u] & kSrcCoded) ? cbase : (fl[u] & kSrcWork) ? wbase : ibase;
        // an asm volatile load: rows of earlier levels are written by the previous grid; an
        // invariant __ldg could be hoisted above the griddepcontrol.wait at kernel entry
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(b0 + static_cast<uint64_t>(m) * t));
      }
      const int32_t lim = min(static_cast<int32_t>(kBatch), nb - kk);
#pragma unroll
      for (int32_t u = 0; u < static_cast<int32_t>(kBatch); ++u) {
        if (u >= lim) break;
        xor_into(acc, v[u]);
        if (fl[u] & kSrcLast) {  // warp-uniform: row complete
          const uint32_t f = static_cast<uint32_t>(__shfl_sync(0xffffffffu, tg, cur));
          uint8_t *ob = (f & kSrcCoded) ? cobase : (f & kSrcWork) ? wobase : obase;
          if (active) *reinterpret_cast<uint4 *>(ob + static_cast<uint64_t>(f & kSrcIndex) * t) = acc;
          acc = make_uint4(0, 0, 0, 0);
          ++cur;
        }
      }
    }
  }
}

// Levels of long rows (late decode levels, repair / update rows: tens to hundreds of sources):
// in fsb_dpg_level a warp walks a row's sources one 512-B gather after another, a serial chain
// of L2 / HBM round trips.  Here a warp covers a 128-B band of its rows as four 8-lane groups:
// group g gathers sources g, g+4, g+8, ... of the row (each group load is one full 128-B line),
// so one load instruction fetches four different sources, and the groups' partial XORs are
// combined by two shuffles.  Units are (stripe, 128-B band, chunk of rows), rows one at a time.
template <uint32_t kBatch, int kMinBlocks>
__global__ void __launch_bounds__(kGlobalThreads, kMinBlocks)
    fsb_dpg_level_q(uint32_t S, uint32_t t, uint32_t nbands, uint32_t row0, uint32_t nrows, uint32_t band_rows,
                    const int32_t *__restrict__ target, const int32_t *__restrict__ src_ptr,
                    const uint32_t *__restrict__ src, uint8_t *coded, uint64_t coded_stride, uint8_t *inter,
                    uint64_t inter_stride, uint8_t *work, uint64_t work_stride, uint32_t rev) {
  static_assert(kBatch == 1 || kBatch == 2 || kBatch == 4 || kBatch == 8, "4 groups x kBatch must divide 32");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t lane = threadIdx.x & 31, grp = lane >> 3;
  const uint32_t nchunks = (nrows + band_rows - 1) / band_rows;
  const uint64_t total = static_cast<uint64_t>(S) * nbands * nchunks;
  uint64_t unit = static_cast<uint64_t>(blockIdx.x) * (kGlobalThreads / 32) + (threadIdx.x >> 5);
  if (unit >= total) return;
  if (rev) unit = total - 1 - unit;
  const uint32_t chunk = static_cast<uint32_t>(unit % nchunks);
  unit /= nchunks;
  const uint32_t band = static_cast<uint32_t>(unit % nbands);
  const uint64_t s = unit / nbands;
  const uint32_t byte_raw = band * kQBandBytes + (lane & 7) * 16;
  const bool active = byte_raw < t;
  const uint32_t byte = active ? byte_raw : 0;
  const uint8_t *ibase = inter + s * inter_stride + byte;
  const uint8_t *cbase = coded + s * coded_stride + byte;
  const uint8_t *wbase = work + s * work_stride + byte;
  const uint32_t r0 = row0 + chunk * band_rows;
  const uint32_t rows = min(band_rows, row0 + nrows - r0);
  for (uint32_t r = r0; r < r0 + rows; ++r) {
    const int32_t a = __ldg(&src_ptr[r]), b = __ldg(&src_ptr[r + 1]);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int32_t e0 = a; e0 < b; e0 += 32) {
      const uint32_t cv = e0 + static_cast<int32_t>(lane) < b ? __ldg(&src[e0 + lane]) : kSrcCoded;
      const int32_t nb = min(32, b - e0);
      for (int32_t kk = 0; kk < nb; kk += 4 * kBatch) {
        uint4 v[kBatch];
#pragma unroll
        for (uint32_t u = 0; u < kBatch; ++u) {
          const int32_t pos = kk + 4 * static_cast<int32_t>(u) + static_cast<int32_t>(grp);
          const uint32_t f = __shfl_sync(0xffffffffu, cv, pos & 31);
          const uint32_t m = f & kSrcIndex;
          const uint8_t *b0 = (f & kSrcCoded) ? cbase : (f & kSrcWork) ? wbase : ibase;
          v[u] = make_uint4(0, 0, 0, 0);
          if (pos < nb)  // (group-uniform) past the row's end: nothing to gather
            asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(b0 + static_cast<uint64_t>(m) * t));
        }
#pragma unroll
        for (uint32_t u = 0; u < kBatch; ++u) xor_into(acc, v[u]);
      }
    }
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
      acc.x ^= __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z ^= __shfl_xor_sync(0xffffffffu, acc.z, o);
      acc.w ^= __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    if (grp == 0 && active) {
      const uint32_t f = static_cast<uint32_t>(__ldg(&target[r]));
      uint8_t *ob = (f & kSrcCoded) ? coded + s * coded_stride : (f & kSrcWork) ? work + s * work_stride
                                                                                : inter + s * inter_stride;
      *reinterpret_cast<uint4 *>(ob + static_cast<uint64_t>(f & kSrcIndex) * t + byte_raw) = acc;
    }
  }
}

// ===================================================================== host-side launch
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

fs_status cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FS_ECUDA;
}

template <typename T>
fs_status upload(T **dst, const T *src, size_t count) {
  *dst = nullptr;
  if (count == 0) return FS_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(dst), count * sizeof(T));
  if (e != cudaSuccess) {
    *dst = nullptr;
    set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return FS_ENOMEM;
  }
  e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
  return FS_OK;
}

}  // namespace

void free_device(Graph &g) {
  DeviceBufs &d = g.dev;
  if (d.device < 0) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(d.device);
  cudaFree(d.pre_row_ptr);
  cudaFree(d.pre_col);
  cudaFree(d.lt_row_ptr);
  cudaFree(d.lt_col);
  cudaFree(d.lt_colf);
  cudaFree(d.win_hdr);
  cudaFree(d.win_ent);
  cudaFree(d.sched);
  cudaFree(d.warp_info);
  cudaFree(d.pre_slots);
  cudaFree(d.pre_level_ptr);
  if (prev >= 0) cudaSetDevice(prev);
  d = DeviceBufs();
}

fs_status upload_graph(Graph &g) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  g.dev.device = dev;
  if ((e = cudaDeviceGetAttribute(&g.sm_count, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  if ((e = cudaDeviceGetAttribute(&g.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  fs_status st;
  if ((st = upload(&g.dev.pre_row_ptr, g.pre_row_ptr.data(), g.pre_row_ptr.size())) != FS_OK) return st;
  if ((st = upload(&g.dev.pre_col, g.pre_col.data(), g.pre_col.size())) != FS_OK) return st;
  if ((st = upload(&g.dev.lt_row_ptr, g.lt_row_ptr.data(), g.lt_row_ptr.size())) != FS_OK) return st;
  if ((st = upload(&g.dev.lt_col, g.lt_col.data(), g.lt_col.size())) != FS_OK) return st;
  {  // column indices marked with the last edge of each row (bit 31), for fsb_lt_band
    std::vector<uint32_t> colf(g.lt_col.begin(), g.lt_col.end());
    for (uint32_t j = 0; j < g.prm.n; ++j) colf[g.lt_row_ptr[j + 1] - 1] |= 0x80000000u;
    if ((st = upload(&g.dev.lt_colf, colf.data(), colf.size())) != FS_OK) return st;
  }
  if (g.win.count) {  // fixed-size edge windows for fsb_lt_win (built on the host, fs_graph_create)
    if ((st = upload(&g.dev.win_hdr, g.win.hdr.data(), g.win.hdr.size())) != FS_OK) return st;
    if ((st = upload(&g.dev.win_ent, g.win.ent.data(), g.win.ent.size())) != FS_OK) return st;
  }
  if (g.smem_eligible) {
    // two tile buffers + the schedule + the precode member rows + 6 mbarriers
    const uint64_t bytes = 2ull * g.sched.tile_units * kUnitBytes + g.sched.words.size() * 4 +
                           ((g.sched.pre_slots.size() * 2 + 15) & ~15ull) + 7 * 8;
    g.smem_bytes = static_cast<uint32_t>(bytes);
    if (bytes > static_cast<uint64_t>(g.smem_optin)) {
      g.smem_eligible = false;
    } else {
      if ((st = upload(&g.dev.sched, g.sched.words.data(), g.sched.words.size())) != FS_OK) return st;
      if ((st = upload(&g.dev.warp_info, g.sched.warp_info.data(), g.sched.warp_info.size())) != FS_OK) return st;
      if ((st = upload(&g.dev.pre_slots, g.sched.pre_slots.data(), g.sched.pre_slots.size())) != FS_OK) return st;
      if ((st = upload(&g.dev.pre_level_ptr, g.pre_level_ptr.data(), g.pre_level_ptr.size())) != FS_OK) return st;
      const int sb = static_cast<int>(g.smem_bytes);
      e = cudaFuncSetAttribute(fsb_smem_encode<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fsb_smem_encode<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fsb_smem_encode<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fsb_smem_encode<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    }
  }
  return FS_OK;
}

// Odd plan levels sweep their (stripe, band) units backwards (FSB_SERPENTINE=0 disables).
static bool serpentine() {
  static const int v = [] {
    const char *e = std::getenv("FSB_SERPENTINE");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// Programmatic dependent launch between dependent kernels of one call (FSB_PDL=0 disables).
static bool pdl_enabled() {
  static const int v = [] {
    const char *e = std::getenv("FSB_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

fs_status launch_encode(const Graph &g, uint32_t S, const uint8_t *data, uint64_t data_stride, uint8_t *checks,
                        uint64_t checks_stride, uint8_t *coded, uint64_t coded_stride, uint32_t row_begin,
                        uint32_t row_end, uint64_t col_begin, uint64_t col_end, void *stream_ptr, uint32_t *launches) {
  *launches = 0;
  const fs_params &prm = g.prm;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g.dev.device) {
      set_error("the graph lives on device " + std::to_string(g.dev.device) + ", the current device is " +
                std::to_string(cur));
      return FS_EINVAL;
    }
  }
  // SMEM tiles need the column range on 64-B slice boundaries
  const bool slice_aligned = col_begin % kSliceBytes == 0 && (col_end % kSliceBytes == 0 || col_end == prm.t);
  const uint32_t slice0 = static_cast<uint32_t>(col_begin / kSliceBytes);
  const uint32_t nslices = static_cast<uint32_t>((col_end + kSliceBytes - 1) / kSliceBytes) - slice0;
  const bool full_rows = row_begin == 0 && row_end == prm.n && slice_aligned;
  const uint64_t tiles = static_cast<uint64_t>(S) * nslices;
  bool use_smem = false;
  if (g.variant == FS_VARIANT_SMEM) {
    if (!g.smem_eligible) { set_error("SMEM variant not eligible for this graph"); return FS_EUNSUPPORTED; }
    use_smem = full_rows;  // row ranges always take the GLOBAL path
    if (use_smem && tiles >= (1ull << 31)) { set_error("launch too large for the SMEM variant"); return FS_EINVAL; }
  } else if (g.variant == FS_VARIANT_AUTO) {
    // SMEM whenever it can run the call: even a few tiles beat the band sweep, whose heavy rows
    // are serial chains of L2 round trips (tools/gpu/auto_probe.py: configs 2/4/6/7 with 1-8
    // stripes, 19-30 us vs 48-160 us; a tie only at config 1's 8 tiles)
    use_smem = g.smem_eligible && full_rows && tiles < (1ull << 31);
  }
  if (S == 0 || row_end == row_begin) {
    if (S == 0 || prm.p == 0) return FS_OK;
  }
  cudaError_t e;
  if (use_smem) {
    auto encode = get_encode_tiled();
    if (!encode) { set_error("cuTensorMapEncodeTiled unavailable"); return FS_ECUDA; }
    CUtensorMap tmap;
    const cuuint64_t dims[3] = {prm.t, prm.k, S};
    const cuuint64_t strides[2] = {prm.t, data_stride};
    const cuuint32_t box[3] = {kSliceBytes, kUnitRows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(data), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) + ")");
      return FS_ECUDA;
    }
    SmemArgs a;
    a.sched = reinterpret_cast<const uint4 *>(g.dev.sched);
    a.warp_info = g.dev.warp_info;
    a.pre_slots = g.dev.pre_slots;
    a.pre_level_ptr = g.dev.pre_level_ptr;
    a.pre_levels = static_cast<uint32_t>(g.pre_level_ptr.size() - 1);
    a.checks = checks;
    a.checks_stride = checks_stride;
    a.coded = coded;
    a.coded_stride = coded_stride;
    a.t = prm.t;
    a.nslices = nslices;
    a.slice0 = slice0;
    a.ntiles = static_cast<uint32_t>(tiles);
    a.p = prm.p;
    a.d_p = prm.d_p;
    a.kpad = g.sched.kpad;
    a.zero_even = g.sched.zero_even;
    a.data_units = g.sched.data_units;
    a.tile_units = g.sched.tile_units;
    a.sched_chunks = static_cast<uint32_t>(g.sched.words.size() / (kChunkBytes / 4));
    // paired tiles (adjacent 64-B slices of a stripe back to back, rows leave as full 128-B lines
    // via TMEM): even slice count and start, and the warps' TMEM column blocks fit one lane quarter
    bool tmem_heads = false;
    {
      static const int paired_env = [] {
        const char *e = std::getenv("FSB_PAIRED");
        return e ? std::atoi(e) : 1;
      }();
      // TMEM columns per lane quarter: 8 per item for the parked results, 8 more per item when the
      // head chunks fit there too (FSB_TMEM_HEADS=0: never, tuning)
      static const int heads_env = [] {
        const char *e = std::getenv("FSB_TMEM_HEADS");
        return e ? std::atoi(e) : 1;
      }();
      uint32_t need = 0;
      for (int q = 0; q < 4; ++q) {
        uint32_t c = 0;
        for (int w = q; w < static_cast<int>(g.sched.nconsumer); w += 4) c += 8 * g.sched.warp_info[w * 3 + 0];
        need = std::max(need, c);
      }
      tmem_heads = heads_env && 2 * need <= 512;
      if (tmem_heads) need *= 2;
      uint32_t cols = 32;
      while (cols < need) cols <<= 1;
      // ... and only when there are more tiles than SMs: a call of at most one tile per SM
      // finishes in one tile time unpaired but two paired (config 2, 64 tiles: 24.7 -> 18.6 us,
      // config 1: 11.2 -> 9.9 us).  FSB_PAIRED=2 pairs regardless (tests), 0 never.
      a.paired = paired_env && nslices % 2 == 0 && slice0 % 2 == 0 && cols <= 512 &&
                 (paired_env == 2 || tiles > static_cast<uint64_t>(g.sm_count));
      a.tmem_cols = cols;
    }
    a.cont_base = g.sched.cont_base;
    a.nc = g.sched.nconsumer;
    {
      // FSB_DEBUG experiments (1 = no TMA loads: wrong bytes by design; 2 = wait counters) exist
      // only in experiment builds (-DFSB_EXPERIMENTS); a release build never reads the variable
#ifdef FSB_EXPERIMENTS
      static const uint32_t dbg = [] {
        const char *e = std::getenv("FSB_DEBUG");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
      }();
      a.debug = dbg;
#else
      a.debug = 0;
#endif
      static const uint32_t wns = [] {
        const char *e = std::getenv("FSB_WAIT_NS");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
      }();
      a.wait_ns = wns;
    }
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(a.paired ? tiles / 2 : tiles, g.sm_count));
    a.pair_tiles = a.tail_tiles = 0;
    if (a.paired) {
      // pair rounds: every CTA gets npairs / grid pairs; a last partial round of R pairs runs as 2R
      // single tiles when they fit one per CTA (2R <= grid), otherwise as pairs (ceil)
      static const int tail_env = [] {
        const char *e = std::getenv("FSB_TAIL_SINGLES");
        return e ? std::atoi(e) : 1;
      }();
      const uint64_t npairs = tiles / 2, jfull = npairs / grid, rem = npairs % grid;
      if (tail_env && rem && 2 * rem <= grid) {
        a.pair_tiles = static_cast<uint32_t>(2 * jfull);
        a.tail_tiles = static_cast<uint32_t>(2 * rem);
      } else {
        a.pair_tiles = static_cast<uint32_t>(2 * ((npairs + grid - 1) / grid));
      }
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = g.smem_bytes;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = pdl_enabled() ? 1 : 0;  // the prologue may overlap the previous grid's tail
    const bool st256 = reinterpret_cast<uintptr_t>(coded) % 32 == 0 && coded_stride % 32 == 0;
    tmem_heads = tmem_heads && a.paired;
    if (st256)
      e = tmem_heads ? cudaLaunchKernelEx(&lc, fsb_smem_encode<true, true>, tmap, a)
                     : cudaLaunchKernelEx(&lc, fsb_smem_encode<true, false>, tmap, a);
    else
      e = tmem_heads ? cudaLaunchKernelEx(&lc, fsb_smem_encode<false, true>, tmap, a)
                     : cudaLaunchKernelEx(&lc, fsb_smem_encode<false, false>, tmap, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fsb_smem_encode launch");
    *launches = 1;
    return FS_OK;
  }
  const uint32_t gslices = static_cast<uint32_t>((col_end - col_begin + kGSliceBytes - 1) / kGSliceBytes);
  for (size_t L = 0; prm.p && L + 1 < g.pre_level_ptr.size(); ++L) {  // one launch per precode level
    const uint32_t c0 = g.pre_level_ptr[L], nc = g.pre_level_ptr[L + 1] - c0;
    const uint64_t items = static_cast<uint64_t>(S) * nc * gslices;
    const uint64_t blocks = (items + kGroupsPerBlock - 1) / kGroupsPerBlock;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(static_cast<uint32_t>(blocks));
    lc.blockDim = dim3(kGlobalThreads);
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = pdl_enabled() && L > 0 ? 1 : 0;  // level L reads the checks of level L-1
    e = cudaLaunchKernelEx(&lc, fsb_precode_global, S, c0, nc, prm.k, prm.d_p, prm.t, col_begin, col_end, gslices,
                           static_cast<const int32_t *>(g.dev.pre_col), data, data_stride, checks, checks_stride);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fsb_precode_global launch");
    ++*launches;
  }
  const uint32_t nrows = row_end - row_begin;
  if (nrows) {
    const uint32_t nbands = static_cast<uint32_t>((col_end - col_begin + kBandBytes - 1) / kBandBytes);
    // rows per warp: up to kBandRowsMax (FSB_BAND_ROWS overrides: tuning experiments), fewer if
    // that leaves fewer than ~64 warps per SM
    static const uint32_t band_rows_max = [] {
      const char *e = std::getenv("FSB_BAND_ROWS");
      return e ? static_cast<uint32_t>(std::atoi(e)) : kBandRowsMax;
    }();
    const uint64_t row_bands = static_cast<uint64_t>(S) * nbands * nrows;
    const uint32_t band_rows = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(band_rows_max, row_bands / (64ull * g.sm_count))));
    const uint64_t units = static_cast<uint64_t>(S) * nbands * ((nrows + band_rows - 1) / band_rows);
    const uint64_t blocks = (units + kGlobalThreads / 32 - 1) / (kGlobalThreads / 32);
    if (blocks >= (1ull << 31)) { set_error("launch too large"); return FS_EINVAL; }
    // Every call whose rows fit the edge windows takes fsb_lt_win: the edges packed into fixed-size
    // windows, 4 gathers per batch, 2-warp blocks, 48 warps per SM (same-box A/B, profiles/r02:
    // config 5 0.221 ms vs 0.251 for fsb_lt_band4 and 0.278 for the round-1 fsb_lt_band<2, 8>;
    // config 3, a few-wave call that ends on its heaviest rows' serial gather chains, 21.6 vs
    // 30.0 us for fsb_lt_band<4, 6, lazy>).  Without windows (a row of more than 93 edges):
    // fsb_lt_band4 for many-wave calls, fsb_lt_band<4, 6, lazy> for few-wave ones.  FSB_BAND_CFG:
    // 5 = this rule (default), 4 = never windows, 1 = fsb_lt_band<2, 8> for every call (the
    // round-1 many-wave kernel), 0 = always <4, 6>, 2 = always <8, 4>.
    static const int band_cfg = [] {
      const char *e = std::getenv("FSB_BAND_CFG");
      return e ? std::atoi(e) : 5;
    }();
    const bool few_waves = units < 4ull * g.sm_count * 64;
    const bool use_win = g.win.count && band_cfg == 5;
    auto kern = fsb_lt_band<4, 6, true>;
    if (band_cfg == 1) kern = fsb_lt_band<2, 8, false>;
    if (band_cfg == 2) kern = fsb_lt_band<8, 4, false>;
    uint64_t blocks_launch = blocks;
    uint32_t block_threads = kGlobalThreads;
    if ((band_cfg == 4 || band_cfg == 5) && !few_waves && !use_win) {
      kern = fsb_lt_band4<4, 24, kBand4Threads>;
      block_threads = kBand4Threads;
      blocks_launch = (units + kBand4Threads / 32 - 1) / (kBand4Threads / 32);
    }
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = pdl_enabled() && prm.p ? 1 : 0;  // overlaps the precode launch
    lc.stream = stream;
    if (use_win) {
      // fixed-size edge windows: the windows holding rows [row_begin, row_end)
      const uint32_t *hw = g.win.hdr.data();
      uint32_t lo = 0, hi = g.win.count;  // last window whose first row <= row_begin
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (hw[2 * mid] <= row_begin) lo = mid; else hi = mid;
      }
      const uint32_t w0 = lo;
      lo = w0; hi = g.win.count;           // last window whose first row < row_end
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (hw[2 * mid] < row_end) lo = mid; else hi = mid;
      }
      const uint32_t nwin = lo + 1 - w0;
      const uint64_t wunits = static_cast<uint64_t>(S) * nbands * nwin;
      const uint64_t wblocks = (wunits + kBand4Threads / 32 - 1) / (kBand4Threads / 32);
      if (wblocks >= (1ull << 31)) { set_error("launch too large"); return FS_EINVAL; }
      lc.gridDim = dim3(static_cast<uint32_t>(wblocks));
      lc.blockDim = dim3(kBand4Threads);
      // full-row calls store every row (no range predicate: one register less, no spill)
      const bool full = row_begin == 0 && row_end == prm.n;
      auto wk = full ? fsb_lt_win<3, 24, kBand4Threads, false> : fsb_lt_win<3, 24, kBand4Threads, true>;
      if (g.win.entries == 128)
        wk = full ? fsb_lt_win<4, 20, kBand4Threads, false> : fsb_lt_win<4, 20, kBand4Threads, true>;
      if (g.win.entries == 160)
        wk = full ? fsb_lt_win<5, 20, kBand4Threads, false> : fsb_lt_win<5, 20, kBand4Threads, true>;
      e = cudaLaunchKernelEx(&lc, wk, S, prm.k, static_cast<uint32_t>(prm.t),
                             static_cast<uint32_t>(col_begin), static_cast<uint32_t>(col_end), nbands, w0, nwin,
                             row_begin, row_end, reinterpret_cast<const uint2 *>(g.dev.win_hdr),
                             static_cast<const uint32_t *>(g.dev.win_ent), data, data_stride,
                             static_cast<const uint8_t *>(checks), checks_stride, coded, coded_stride);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "fsb_lt_win launch");
      ++*launches;
      return FS_OK;
    }
    lc.gridDim = dim3(static_cast<uint32_t>(blocks_launch));
    lc.blockDim = dim3(block_threads);
    e = cudaLaunchKernelEx(&lc, kern, S, prm.k, static_cast<uint32_t>(prm.t), static_cast<uint32_t>(col_begin),
                           static_cast<uint32_t>(col_end), nbands, row_begin, nrows, band_rows,
                           static_cast<const int32_t *>(g.dev.lt_row_ptr), static_cast<const uint32_t *>(g.dev.lt_colf),
                           data, data_stride, static_cast<const uint8_t *>(checks), checks_stride, coded,
                           coded_stride);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fsb_lt_band launch");
    ++*launches;
  }
  return FS_OK;
}

struct PlanGraphCache {
  std::mutex mu;
  cudaStream_t cap = nullptr;          // private stream the levels are captured on
  cudaGraphExec_t exec = nullptr;
  uint32_t S = 0, launches = 0;
  const void *coded = nullptr, *inter = nullptr;
  uint64_t coded_stride = 0, inter_stride = 0;
  uint8_t *work = nullptr;             // workspace rows (inactivation decoding), grown on demand
  uint64_t work_bytes = 0;
  ~PlanGraphCache() {
    if (exec) cudaGraphExecDestroy(exec);
    if (cap) cudaStreamDestroy(cap);
    if (work) cudaFree(work);
  }
};

fs_status upload_decode_plan(DecodePlan &pl) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  pl.device = dev;
  if ((e = cudaDeviceGetAttribute(&pl.sm_count, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  fs_status st;
  if ((st = upload(&pl.d_target, pl.target.data(), pl.target.size())) != FS_OK) return st;
  if ((st = upload(&pl.d_src_ptr, pl.src_ptr.data(), pl.src_ptr.size())) != FS_OK) return st;
  if ((st = upload(&pl.d_src, pl.src.data(), pl.src.size())) != FS_OK) return st;
  pl.gcache = std::make_shared<PlanGraphCache>();
  return FS_OK;
}

void free_decode_plan(DecodePlan &pl) {
  if (pl.device < 0) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(pl.device);
  cudaFree(pl.d_target);
  cudaFree(pl.d_src_ptr);
  cudaFree(pl.d_src);
  pl.gcache.reset();  // graph exec and capture stream of this device
  if (prev >= 0) cudaSetDevice(prev);
  pl.d_target = pl.d_src_ptr = nullptr;
  pl.d_src = nullptr;
  pl.device = -1;
}

fs_status launch_decode(const DecodePlan &pl, uint32_t S, const uint8_t *coded, uint64_t coded_stride,
                        uint8_t *inter, uint64_t inter_stride, void *stream_ptr, uint32_t *launches) {
  // decode plans never target coded rows, so the coded buffer is only read
  return launch_plan(pl, S, const_cast<uint8_t *>(coded), coded_stride, inter, inter_stride, stream_ptr, launches);
}

static fs_status launch_levels(const DecodePlan &pl, uint32_t S, uint8_t *coded, uint64_t coded_stride,
                               uint8_t *inter, uint64_t inter_stride, uint8_t *work, uint64_t work_stride,
                               cudaStream_t stream, uint32_t *launches);

// Plans with several levels replay a CUDA graph of their level launches (captured on first use
// for these buffers), so the ~1.5 us launch gap between dependent levels goes away;
// FSB_GRAPH=0 launches level by level.
fs_status launch_plan(const DecodePlan &pl, uint32_t S, uint8_t *coded, uint64_t coded_stride,
                      uint8_t *inter, uint64_t inter_stride, void *stream_ptr, uint32_t *launches) {
  static const int use_graph = [] {
    const char *e = std::getenv("FSB_GRAPH");
    return e ? std::atoi(e) : 1;
  }();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != pl.device) {
      set_error("the plan lives on device " + std::to_string(pl.device) + ", the current device is " +
                std::to_string(cur));
      return FS_EINVAL;
    }
  }
  if (!pl.gcache) return launch_levels(pl, S, coded, coded_stride, inter, inter_stride, nullptr, 0, stream, launches);
  PlanGraphCache &c = *pl.gcache;
  std::lock_guard<std::mutex> lock(c.mu);
  cudaError_t e;
  // workspace for the plan's Z rows: work_rows x t per stripe (allocated once, grown if needed)
  const uint64_t work_stride = static_cast<uint64_t>(pl.work_rows) * pl.t;
  const uint64_t need = work_stride * S;
  if (need > c.work_bytes) {
    if (c.work) {
      cudaStreamSynchronize(stream);  // a replayed graph may still read the old buffer
      cudaFree(c.work);
      c.work = nullptr;
      c.work_bytes = 0;
      if (c.exec) {
        cudaGraphExecDestroy(c.exec);
        c.exec = nullptr;
      }
    }
    if ((e = cudaMalloc(&c.work, need)) != cudaSuccess) return cuda_fail(e, "cudaMalloc (decode workspace)");
    c.work_bytes = need;
  }
  if (!use_graph || pl.level_ptr.size() < 3)
    return launch_levels(pl, S, coded, coded_stride, inter, inter_stride, c.work, work_stride, stream, launches);
  if (!c.exec || c.S != S || c.coded != coded || c.inter != inter || c.coded_stride != coded_stride ||
      c.inter_stride != inter_stride) {
    if (c.exec) {
      cudaGraphExecDestroy(c.exec);
      c.exec = nullptr;
    }
    if (!c.cap && (e = cudaStreamCreateWithFlags(&c.cap, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreateWithFlags");
    if ((e = cudaStreamBeginCapture(c.cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamBeginCapture");
    uint32_t n = 0;
    fs_status st = launch_levels(pl, S, coded, coded_stride, inter, inter_stride, c.work, work_stride, c.cap, &n);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(c.cap, &graph);
    if (st != FS_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&c.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      c.exec = nullptr;
      return cuda_fail(e, "cudaGraphInstantiate");
    }
    c.S = S, c.coded = coded, c.inter = inter, c.coded_stride = coded_stride, c.inter_stride = inter_stride;
    c.launches = n;
  }
  if ((e = cudaGraphLaunch(c.exec, stream)) != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
  *launches = c.launches;
  return FS_OK;
}

// rows per unit of a level: as many as keep >= 64 warps' worth of units per SM (1..8)
static uint32_t level_band_rows(uint64_t row_bands, int sm_count) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kBandRowsMax, row_bands / (64ull * sm_count))));
}

static fs_status launch_levels(const DecodePlan &pl, uint32_t S, uint8_t *coded, uint64_t coded_stride,
                               uint8_t *inter, uint64_t inter_stride, uint8_t *work, uint64_t work_stride,
                               cudaStream_t stream, uint32_t *launches) {
  *launches = 0;
  const uint32_t nbands = static_cast<uint32_t>((pl.t + kBandBytes - 1) / kBandBytes);
  for (size_t L = 0; L + 1 < pl.level_ptr.size(); ++L) {
    const uint32_t row0 = pl.level_ptr[L], nrows = pl.level_ptr[L + 1] - row0;
    if (!nrows) continue;
    const uint64_t row_bands = static_cast<uint64_t>(S) * nbands * nrows;
    const uint32_t band_rows = level_band_rows(row_bands, pl.sm_count);
    const uint64_t units = static_cast<uint64_t>(S) * nbands * ((nrows + band_rows - 1) / band_rows);
    // gathers in flight per warp: levels of long rows (repair / update / dense decode levels) take 8
    // at 4 blocks per SM, levels of short rows 2 at 6 blocks (measured on configs 5, 7 and 4:
    // update 3.41 -> 3.10 ms, repair 0.457 -> 0.384, decode 0.722 -> 0.687 with 8 in flight; the
    // 86 small levels of the config-4 inactivation decode prefer 2).  FSB_DPG_CFG=1/2 forces one.
    static const int dpg_cfg = [] {
      const char *e = std::getenv("FSB_DPG_CFG");
      return e ? std::atoi(e) : 0;
    }();
    const uint32_t nsrc = static_cast<uint32_t>(pl.src_ptr[row0 + nrows] - pl.src_ptr[row0]);
    const bool long_rows = dpg_cfg == 2 || (dpg_cfg == 0 && nsrc >= 6u * nrows);
    auto kern = long_rows ? fsb_dpg_level<8, 4> : fsb_dpg_level<2, 6>;
    // Levels of very long rows (>= FSB_DPG_Q sources on average; update: ~234) with enough units
    // for >= 4 waves: four source streams per warp over 128-B bands (fsb_dpg_level_q<4, 6>).
    // Measured (one box, tools/gpu/dpgq_sweep.sh): update 3.11 -> 2.34 ms; it loses where the
    // rows are shorter (decode's late levels, 30-60 sources: 0.655 -> 0.664-0.72 ms) or the level
    // is too small to fill the GPU (repair's 13 rows: 0.384 -> 0.42-0.53 ms).
    static const uint32_t q_min = [] {
      const char *e = std::getenv("FSB_DPG_Q");
      return e ? static_cast<uint32_t>(std::atoi(e)) : 100u;
    }();
    static const int q_cfg = [] {
      const char *e = std::getenv("FSB_DPG_QCFG");
      return e ? std::atoi(e) : 1;
    }();
    static const int q_rows = [] {
      const char *e = std::getenv("FSB_DPG_QROWS");
      return e ? std::atoi(e) : 0;
    }();
    uint32_t nb = nbands, br = band_rows;
    uint64_t nunits = units;
    if (q_min && nsrc >= static_cast<uint64_t>(q_min) * nrows) {
      const uint32_t qnb = static_cast<uint32_t>((pl.t + kQBandBytes - 1) / kQBandBytes);
      const uint32_t qbr = q_rows > 0 ? std::min<uint32_t>(kBandRowsMax, static_cast<uint32_t>(q_rows))
                                      : level_band_rows(static_cast<uint64_t>(S) * qnb * nrows, pl.sm_count);
      const uint64_t qunits = static_cast<uint64_t>(S) * qnb * ((nrows + qbr - 1) / qbr);
      if (q_min == 1 || qunits >= 4ull * pl.sm_count * 48) {  // FSB_DPG_Q=1: every level (tests)
        kern = q_cfg == 0 ? fsb_dpg_level_q<8, 4> : q_cfg == 2 ? fsb_dpg_level_q<2, 8> : fsb_dpg_level_q<4, 6>;
        nb = qnb, br = qbr, nunits = qunits;
      }
    }
    const uint64_t blocks = (nunits + kGlobalThreads / 32 - 1) / (kGlobalThreads / 32);
    if (blocks >= (1ull << 31)) { set_error("launch too large"); return FS_EINVAL; }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(static_cast<uint32_t>(blocks));
    lc.blockDim = dim3(kGlobalThreads);
    lc.dynamicSmemBytes = 0;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = pdl_enabled() && L > 0 ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&lc, kern, S, static_cast<uint32_t>(pl.t), nb, row0, nrows, br,
                                       static_cast<const int32_t *>(pl.d_target),
                                       static_cast<const int32_t *>(pl.d_src_ptr),
                                       static_cast<const uint32_t *>(pl.d_src), coded, coded_stride, inter,
                                       inter_stride, work, work_stride, serpentine() ? static_cast<uint32_t>(L & 1) : 0u);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fsb_dpg_level launch");
    ++*launches;
  }
  return FS_OK;
}

fs_status read_debug_counters(uint64_t *out, uint32_t n) {
  static unsigned long long buf[kDebugCounters];
  cudaError_t e = cudaMemcpyFromSymbol(buf, g_debug_counters, sizeof(buf));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyFromSymbol");
  for (uint32_t i = 0; i < n && i < kDebugCounters; ++i) out[i] = buf[i];
  static const unsigned long long zero[kDebugCounters] = {0};
  e = cudaMemcpyToSymbol(g_debug_counters, zero, sizeof(zero));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyToSymbol");
  return FS_OK;
}

}  // namespace fsb
