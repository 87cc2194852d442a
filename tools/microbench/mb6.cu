// Coded-row store paths for the SMEM kernel's item epilogue (8 rows x 64 B per warp per item):
//   V=0  STG: every half-group stores its 64 B (8 distinct 128-B lines per store)
//   V=1  staged TMA scatter: each half-group writes its 64 B to a per-warp staging slot (STS),
//        lane 0 issues two cp.async.bulk.tensor.2d ... tile::scatter4 ops (rows 0-3, 4-7),
//        staging double-buffered with cp.async.bulk.wait_group.read
// interleaved with parity-paired 64-B gathers (GATHERS per item).  Prints clk per item per SM.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

constexpr int ROWS = 2048, GATHERS = 10;

template <int V>
__global__ void __launch_bounds__(512, 1) epi(const __grid_constant__ CUtensorMap tm, uint4* out, int iters) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint4* sm = reinterpret_cast<uint4*>(smem);
  uint8_t* stage = smem + ROWS * 64;                 // 16 warps x 2 buffers x 512 B
  for (int i = threadIdx.x; i < ROWS * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1, w = threadIdx.x >> 5;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  uint32_t hw = (blockIdx.x * 4096 + w) * 2654435761u;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < GATHERS; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (ROWS - 1), rb = (h >> 20) & (ROWS - 1);
      uint32_t r = half ? (rb | 1) : (ra & ~1u);
      uint4 v = sm[r * 4 + lane4];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    hw = hw * 1664525u + 1013904223u;
    const uint32_t hg = lane >> 2;
    const uint32_t row = (hw + hg * 7919u) & 2047u;
    if (V == 0) {
      out[row * 256 + blockIdx.x * 4 + lane4] = acc;
    } else {
      const uint32_t buf = it & 1;
      uint8_t* slot = stage + (w * 2 + buf) * 512;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      *reinterpret_cast<uint4*>(slot + hg * 64 + lane4 * 16) = acc;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      uint32_t rr[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) rr[q] = __shfl_sync(0xffffffffu, row, q * 4);
      if (lane == 0) {
        const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(slot));
        const int32_t x = blockIdx.x * 64;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     :: "l"(&tm), "r"(x), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(s0) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     :: "l"(&tm), "r"(x), "r"(rr[4]), "r"(rr[5]), "r"(rr[6]), "r"(rr[7]), "r"(s0 + 256) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (V == 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // output: 2048 rows x 16 KB (row stride 16384 B), enough columns for 148 CTAs x 64 B... use 256 uint4 = 4 KB per row
  uint4* out; cudaMalloc(&out, (size_t)2048 * 4096 * 4);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4096 * 4, 2048};          // bytes per row (>= 148*64), rows
  cuuint64_t strides[1] = {4096 * 4};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, out, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int smem = ROWS * 64 + 16 * 2 * 512, iters = 4096;
  cudaFuncSetAttribute(epi<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(epi<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (v == 0) epi<0><<<sms, 512, smem>>>(tm, out, iters); else epi<1><<<sms, 512, smem>>>(tm, out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      printf("{\"variant\":%d,\"ms\":%.4f,\"clk_per_item_per_sm\":%.2f,\"err\":\"%s\"}\n", v, ms,
             ms * 1e-3 * clk * 1e3 / (16.0 * iters), cudaGetErrorString(e));
    }
  }
  return 0;
}
