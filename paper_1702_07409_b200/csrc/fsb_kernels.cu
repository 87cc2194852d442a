// sm_100a kernels of the Founsure encode path (§2.2 steps (1) and (2)).
//
//   precode   C_i = XOR_{m in P(i)} D_m              (a3)
//   LT        Y_j = XOR_{m in N(j)} I_m, I = D ++ C   (a4)
//   stripes   the same graph over every stripe       (a5)
//
// Two variants, bit-identical output (XOR is exact and order-free):
//
// SMEM  (fsb_smem_encode): persistent, one CTA per SM.  A tile = (stripe, 128-byte slice of
//       every symbol).  A TMA producer warp streams the tile's k data rows (32 rows x 128 B
//       per cp.async.bulk.tensor box) into a shared-memory ring; 16 consumer warps compute
//       the p checks from shared memory (written back to smem and HBM), then every coded
//       row as a register XOR of 16-B lanes gathered from shared memory, and store it with
//       one full 128-B line per row.  HBM sees each source byte once and each output byte
//       once (the ideal one-read-one-write roofline); the gathers hit shared memory only.
//       Tiles alternate between the two ends of the ring so the next tile's rows stream in
//       while the current one computes.  Work per warp comes from a host-built, degree-
//       aware schedule (fsb_graph.cpp): heavy rows are split over the 4 lane-groups of a
//       warp and recombined with shuffles; light rows are packed by equal degree.
//
// GLOBAL (fsb_precode_global + fsb_lt_global): no staging; every group of 8 lanes XORs one
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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
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

// ============================================================================ SMEM kernel
struct SmemArgs {
  const uint32_t *sched;       // kConsumerWarps x (NR*32) schedule words
  const uint32_t *warp_steps;  // kConsumerWarps
  const uint16_t *pre_slots;   // p * d_p
  uint8_t *checks;
  uint64_t checks_stride;
  uint8_t *coded;
  uint64_t coded_stride;
  uint64_t t;
  uint32_t nslices, ntiles, p, d_p, kpad, data_units, tile_units, ring_units;
};

// Use index of ring unit x by the CTA's i-th tile (even tiles occupy [0,T), odd [U-T,U)).
__device__ __forceinline__ uint32_t unit_use(uint32_t x, uint32_t i, uint32_t T, uint32_t U) {
  const bool in_even = x < T, in_odd = x + T >= U;
  return (in_even && in_odd) ? i : (i >> 1);
}

template <int NR>
__device__ __forceinline__ void store_item(uint4 acc, uint32_t v, uint32_t grp, uint8_t *out, uint64_t t) {
  if (v & kSplitFlag) {  // split row: combine the four groups' partial XORs (uniform branch)
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1) {
      acc.x ^= __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z ^= __shfl_xor_sync(0xffffffffu, acc.z, o);
      acc.w ^= __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    if (grp == 0) st_stream(out + static_cast<uint64_t>(v & 0x3FFF) * t, acc);
  } else if ((v & 0x3FFF) != 0x3FFF) {
    st_stream(out + static_cast<uint64_t>(v & 0x3FFF) * t, acc);
  }
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    fsb_smem_encode(const __grid_constant__ CUtensorMap tmap, const SmemArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t U = a.ring_units, T = a.tile_units;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + static_cast<size_t>(U) * kUnitBytes);
  uint64_t *empty = full + U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (uint32_t x = 0; x < U; ++x) {
      mbar_init(smem_u32(&full[x]), 1);
      mbar_init(smem_u32(&empty[x]), kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t ov = (2 * T > U) ? 2 * T - U : 0;  // units shared by consecutive tiles

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ TMA producer (1 lane)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      const uint64_t pol = policy_evict_first();
      uint32_t i = 0;
      for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++i) {
        const uint32_t stripe = tile / a.nslices, slice = tile % a.nslices;
        const uint32_t base = (i & 1) ? U - T : 0;
        for (uint32_t j = 0; j < T; ++j) {
          // units private to this parity first, the units shared with the previous tile last
          const uint32_t u = (i & 1) ? (j + ov) % T : j;
          const uint32_t x = base + u;
          const uint32_t use = unit_use(x, i, T, U);
          mbar_wait(smem_u32(&empty[x]), (use & 1) ^ 1);
          if (u < a.data_units) {
            mbar_arrive_expect_tx(smem_u32(&full[x]), kUnitBytes);
            tma_load_3d(smem_u32(smem + static_cast<size_t>(x) * kUnitBytes), &tmap, smem_u32(&full[x]),
                        static_cast<int32_t>(slice * kSliceBytes), static_cast<int32_t>(u * kUnitRows),
                        static_cast<int32_t>(stripe), pol);
          } else {
            mbar_arrive(smem_u32(&full[x]));  // check rows: written by the consumers
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------- consumer warps
  const uint4 *ring4 = reinterpret_cast<const uint4 *>(smem);
  uint4 *ring4w = reinterpret_cast<uint4 *>(smem);
  const uint32_t grp = lane >> 3, lane8 = lane & 7;
  const uint32_t gidx = warp * kGroupsPerWarp + grp;
  // this warp's whole LT schedule lives in registers for the kernel's lifetime
  uint32_t R[NR];
  {
    const uint32_t *sw = a.sched + static_cast<size_t>(warp) * (NR * 32);
#pragma unroll
    for (int r = 0; r < NR; ++r) R[r] = __ldg(&sw[r * 32 + lane]);
  }
  const uint32_t nsteps = __ldg(&a.warp_steps[warp]);
  const uint32_t src_hi = grp >> 1, sh = (grp & 1) * 16;
  uint32_t i = 0;
  for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++i) {
    const uint32_t stripe = tile / a.nslices, slice = tile % a.nslices;
    const uint32_t base_unit = (i & 1) ? U - T : 0;
    const uint32_t tbase = base_unit * (kUnitBytes / 16) + lane8;  // uint4 index of row 0, my lane
    for (uint32_t u = 0; u < T; ++u) {
      const uint32_t x = base_unit + u;
      mbar_wait(smem_u32(&full[x]), unit_use(x, i, T, U) & 1);
    }
    const uint64_t col_off = static_cast<uint64_t>(slice) * kSliceBytes + lane8 * 16;

    // (1) precode checks (PAPER.md:91 step (1)): into the tile's check rows and to HBM
    if (a.p) {
      for (uint32_t c = gidx; c < a.p; c += kGroups) {
        uint4 acc = make_uint4(0, 0, 0, 0);
        for (uint32_t e = 0; e < a.d_p; ++e) {
          const uint32_t s = __ldg(&a.pre_slots[c * a.d_p + e]);
          xor_into(acc, ring4[tbase + s * 8]);
        }
        ring4w[tbase + (a.kpad + c) * 8] = acc;
        st_stream(a.checks + stripe * a.checks_stride + c * a.t + col_off, acc);
      }
      consumer_bar();
    }

    // (2) LT rows (PAPER.md:91 step (2)): step e of group grp is a warp shuffle away
    uint8_t *out = a.coded + stripe * a.coded_stride + col_off;
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (static_cast<uint32_t>(r) * kStepsPerReg >= nsteps) break;
      const uint32_t reg = R[r];
      for (uint32_t q = 0; q < static_cast<uint32_t>(kStepsPerReg); q += 4) {
        if (r * kStepsPerReg + q >= nsteps) break;
        uint32_t v[4];
        uint4 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (__shfl_sync(0xffffffffu, reg, 2 * (q + j) + src_hi) >> sh) & 0xFFFF;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          x[j] = make_uint4(0, 0, 0, 0);
          if (v[j] < kIdle) x[j] = ring4[tbase + v[j] * 8];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (v[j] & kStoreFlag) {  // store step: the same for every group of the warp
            store_item<NR>(acc, v[j], grp, out, a.t);
            acc = make_uint4(0, 0, 0, 0);
          } else {
            xor_into(acc, x[j]);
          }
        }
      }
    }
    // release the tile's units to the producer
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      for (uint32_t u = 0; u < T; ++u) mbar_arrive(smem_u32(&empty[base_unit + u]));
    }
  }
}

// ========================================================================= GLOBAL kernels
constexpr int kGlobalThreads = 256;
constexpr int kGroupsPerBlock = kGlobalThreads / 8;
constexpr uint32_t kBandSlices = 4;  // 512-B bands: one warp = one row x 4 slices

__global__ void __launch_bounds__(kGlobalThreads)
    fsb_precode_global(uint32_t S, uint32_t p, uint32_t d_p, uint64_t t, uint32_t nslices,
                       const int32_t *__restrict__ pre_col, const uint8_t *__restrict__ data,
                       uint64_t data_stride, uint8_t *__restrict__ checks, uint64_t checks_stride) {
  const uint64_t item = static_cast<uint64_t>(blockIdx.x) * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint32_t lane8 = threadIdx.x & 7;
  const uint64_t total = static_cast<uint64_t>(S) * p * nslices;
  if (item >= total) return;
  const uint32_t slice = item % nslices;
  const uint64_t r = item / nslices;
  const uint32_t c = r % p;
  const uint32_t s = static_cast<uint32_t>(r / p);
  const uint64_t byte = static_cast<uint64_t>(slice) * kSliceBytes + lane8 * 16;
  if (byte >= t) return;
  const uint8_t *src = data + s * data_stride + byte;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint32_t e = 0; e < d_p; ++e) {
    const int32_t m = __ldg(&pre_col[c * d_p + e]);
    xor_into(acc, __ldg(reinterpret_cast<const uint4 *>(src + static_cast<uint64_t>(m) * t)));
  }
  *reinterpret_cast<uint4 *>(checks + s * checks_stride + static_cast<uint64_t>(c) * t + byte) = acc;
}

__global__ void __launch_bounds__(kGlobalThreads)
    fsb_lt_global(uint32_t S, uint32_t k, uint64_t t, uint32_t nslices, uint32_t nbands,
                  uint32_t row_begin, uint32_t nrows, const int32_t *__restrict__ row_ptr,
                  const int32_t *__restrict__ col, const uint8_t *__restrict__ data, uint64_t data_stride,
                  const uint8_t *__restrict__ checks, uint64_t checks_stride, uint8_t *__restrict__ coded,
                  uint64_t coded_stride) {
  uint64_t e = static_cast<uint64_t>(blockIdx.x) * kGroupsPerBlock + (threadIdx.x >> 3);
  const uint32_t lane8 = threadIdx.x & 7;
  const uint32_t q = e % kBandSlices;
  e /= kBandSlices;
  const uint32_t jr = e % nrows;
  e /= nrows;
  const uint32_t band = e % nbands;
  const uint64_t s = e / nbands;
  if (s >= S) return;
  const uint32_t slice = band * kBandSlices + q;
  const uint64_t byte = static_cast<uint64_t>(slice) * kSliceBytes + lane8 * 16;
  if (slice >= nslices || byte >= t) return;
  const uint32_t j = row_begin + jr;
  const uint8_t *dsrc = data + s * data_stride + byte;
  const uint8_t *csrc = checks + s * checks_stride + byte;
  int32_t b = __ldg(&row_ptr[j]);
  const int32_t end = __ldg(&row_ptr[j + 1]);
  uint4 acc = make_uint4(0, 0, 0, 0);
  auto src = [&](int32_t m) -> const uint4 * {
    return reinterpret_cast<const uint4 *>(static_cast<uint32_t>(m) < k
                                               ? dsrc + static_cast<uint64_t>(m) * t
                                               : csrc + static_cast<uint64_t>(m - k) * t);
  };
  for (; b + 4 <= end; b += 4) {
    const int32_t m0 = __ldg(&col[b]), m1 = __ldg(&col[b + 1]), m2 = __ldg(&col[b + 2]), m3 = __ldg(&col[b + 3]);
    const uint4 v0 = __ldg(src(m0)), v1 = __ldg(src(m1)), v2 = __ldg(src(m2)), v3 = __ldg(src(m3));
    xor_into(acc, v0);
    xor_into(acc, v1);
    xor_into(acc, v2);
    xor_into(acc, v3);
  }
  for (; b < end; ++b) xor_into(acc, __ldg(src(__ldg(&col[b]))));
  st_stream(coded + s * coded_stride + static_cast<uint64_t>(jr) * t + byte, acc);
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
  cudaFree(d.sched);
  cudaFree(d.warp_steps);
  cudaFree(d.pre_slots);
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
  if (g.smem_eligible) {
    // ring size: as many 4-KiB units as the opt-in shared memory allows (barriers after them)
    uint32_t units = static_cast<uint32_t>((g.smem_optin - 1024) / (kUnitBytes + 16));
    if (const char *env = std::getenv("FSB_RING_UNITS")) units = std::min<uint32_t>(units, std::atoi(env));
    g.ring_units = units;
    g.smem_bytes = units * kUnitBytes + units * 16;
    if (g.sched.tile_units > units || g.sched.tile_units == 0) {
      g.smem_eligible = false;
    } else {
      if ((st = upload(&g.dev.sched, g.sched.words.data(), g.sched.words.size())) != FS_OK) return st;
      if ((st = upload(&g.dev.warp_steps, g.sched.warp_steps.data(), g.sched.warp_steps.size())) != FS_OK) return st;
      if ((st = upload(&g.dev.pre_slots, g.sched.pre_slots.data(), g.sched.pre_slots.size())) != FS_OK) return st;
      e = cudaFuncSetAttribute(fsb_smem_encode<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(g.smem_bytes));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fsb_smem_encode<kSchedRegsMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(g.smem_bytes));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    }
  }
  return FS_OK;
}

fs_status launch_encode(const Graph &g, uint32_t S, const uint8_t *data, uint64_t data_stride, uint8_t *checks,
                        uint64_t checks_stride, uint8_t *coded, uint64_t coded_stride, uint32_t row_begin,
                        uint32_t row_end, void *stream_ptr, uint32_t *launches) {
  *launches = 0;
  const fs_params &prm = g.prm;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  const uint32_t nslices = static_cast<uint32_t>((prm.t + kSliceBytes - 1) / kSliceBytes);
  const bool full_rows = row_begin == 0 && row_end == prm.n;
  const uint64_t tiles = static_cast<uint64_t>(S) * nslices;
  bool use_smem = false;
  if (g.variant == FS_VARIANT_SMEM) {
    if (!g.smem_eligible) { set_error("SMEM variant not eligible for this graph"); return FS_EUNSUPPORTED; }
    use_smem = full_rows;  // row ranges always take the GLOBAL path
  } else if (g.variant == FS_VARIANT_AUTO) {
    use_smem = g.smem_eligible && full_rows && tiles >= 2ull * g.sm_count && tiles < (1ull << 31);
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
    a.sched = g.dev.sched;
    a.warp_steps = g.dev.warp_steps;
    a.pre_slots = g.dev.pre_slots;
    a.checks = checks;
    a.checks_stride = checks_stride;
    a.coded = coded;
    a.coded_stride = coded_stride;
    a.t = prm.t;
    a.nslices = nslices;
    a.ntiles = static_cast<uint32_t>(tiles);
    a.p = prm.p;
    a.d_p = prm.d_p;
    a.kpad = g.sched.kpad;
    a.data_units = g.sched.data_units;
    a.tile_units = g.sched.tile_units;
    a.ring_units = g.ring_units;
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(tiles, g.sm_count));
    if (g.sched.regs <= 16)
      fsb_smem_encode<16><<<grid, kThreads, g.smem_bytes, stream>>>(tmap, a);
    else
      fsb_smem_encode<kSchedRegsMax><<<grid, kThreads, g.smem_bytes, stream>>>(tmap, a);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fsb_smem_encode launch");
    *launches = 1;
    return FS_OK;
  }
  if (prm.p) {
    const uint64_t items = static_cast<uint64_t>(S) * prm.p * nslices;
    const uint64_t blocks = (items + kGroupsPerBlock - 1) / kGroupsPerBlock;
    fsb_precode_global<<<static_cast<uint32_t>(blocks), kGlobalThreads, 0, stream>>>(
        S, prm.p, prm.d_p, prm.t, nslices, g.dev.pre_col, data, data_stride, checks, checks_stride);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fsb_precode_global launch");
    ++*launches;
  }
  const uint32_t nrows = row_end - row_begin;
  if (nrows) {
    const uint32_t nbands = (nslices + kBandSlices - 1) / kBandSlices;
    const uint64_t items = static_cast<uint64_t>(S) * nbands * nrows * kBandSlices;
    const uint64_t blocks = (items + kGroupsPerBlock - 1) / kGroupsPerBlock;
    if (blocks >= (1ull << 31)) { set_error("launch too large"); return FS_EINVAL; }
    fsb_lt_global<<<static_cast<uint32_t>(blocks), kGlobalThreads, 0, stream>>>(
        S, prm.k, prm.t, nslices, nbands, row_begin, nrows, g.dev.lt_row_ptr, g.dev.lt_col, data, data_stride,
        checks, checks_stride, coded, coded_stride);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fsb_lt_global launch");
    ++*launches;
  }
  return FS_OK;
}

}  // namespace fsb
