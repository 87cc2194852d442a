// Does tensor memory (TMEM) traffic compete with shared-memory gathers for the L1TEX/LSU pipe?
// Candidate design: park the even tile's 64-B row results in TMEM (tcgen05.st) and, in the odd
// tile (the adjacent 64-B slice of the same stripe), read them back (tcgen05.ld) so every coded
// row leaves as full 128-B lines.  Every variant does the parity-paired 64-B gathers of mb3/mb5
// and adds, per 8 gathers:
//   0: nothing (baseline)
//   1: one tcgen05.st.32x32b.x4 (16 B per lane)
//   2: one tcgen05.ld.32x32b.x4 + tcgen05.wait::ld
//   3: both (st then ld of another column block)
//   6: one half-line STG (8 rows x 64 B per warp store; mb5 variant 6 = today's coded-row store)
//   7: one full-line STG (4 rows x 128 B)
//   9: per 16 gathers: one tcgen05.ld + two full-line STGs (the candidate's odd-tile store path),
//      i.e. per 8 gathers half of that
// Prints clk per warp-gather per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st4(uint32_t taddr, uint4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 tm_ld4(uint32_t taddr) {
  uint4 v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return v;
}

template <int V>
__global__ void __launch_bounds__(512, 1) mix(uint4* out, int rows, int iters) {
  extern __shared__ __align__(128) uint4 sm[];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1;
  // this warp's TMEM: lanes 32*(warp%4).., columns (warp/4)*32 .. +32
  const uint32_t taddr = tbase + ((32u * (warp & 3)) << 16) + (warp >> 2) * 32;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  uint32_t hw = (blockIdx.x * 4096 + warp) * 2654435761u;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
      uint32_t r = half ? (rb | 1) : (ra & ~1u);
      uint4 v = sm[r * 4 + lane4];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    hw = hw * 1664525u + 1013904223u;
    const uint32_t col = (it & 7) * 4;
    if (V == 1 || V == 3) tm_st4(taddr + col, acc);
    if (V == 2 || V == 3) {
      uint4 x = tm_ld4(taddr + ((col + 16) & 31));
      acc.x ^= x.y; acc.y ^= x.x;
    }
    if (V == 6) {
      const uint32_t row = (hw + (threadIdx.x >> 2) * 7919u) & 2047u;
      out[(row * 256 + blockIdx.x * 4 + lane4) & (1024 * 512 - 1)] = acc;
    }
    if (V == 7) {
      const uint32_t row = (hw + (threadIdx.x >> 3) * 7919u) & 2047u;
      out[(row * 256 + blockIdx.x * 8 + (lane & 7)) & (1024 * 512 - 1)] = acc;
    }
    if (V == 9 && (it & 1)) {
      uint4 x = tm_ld4(taddr + col);
      const uint32_t row = (hw + (threadIdx.x >> 3) * 7919u) & 2047u;
      out[(row * 256 + blockIdx.x * 8 + (lane & 7)) & (1024 * 512 - 1)] = acc;
      const uint32_t row2 = (hw * 3 + (threadIdx.x >> 3) * 7919u) & 2047u;
      out[(row2 * 256 + blockIdx.x * 8 + (lane & 7)) & (1024 * 512 - 1)] = x;
    }
    if (V == 9 && !(it & 1)) tm_st4(taddr + ((col + 4) & 31), acc);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase) : "memory");
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(uint4* out, int sms) {
  const int rows = 2048, iters = 2048, threads = 512;
  const size_t smem = rows * 64;
  cudaFuncSetAttribute(mix<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mix<V><<<sms, threads, smem>>>(out, rows, 8);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("variant %d: %s\n", V, cudaGetErrorString(e)); return; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  mix<V><<<sms, threads, smem>>>(out, rows, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double gathers = (double)sms * (threads / 32) * iters * 8;
  printf("{\"variant\":%d,\"ms\":%.4f,\"clk_per_gather_per_sm\":%.3f}\n", V, ms,
         ms * 1e-3 * clk * 1e3 / (gathers / sms));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out; cudaMalloc(&out, 1024 * 512 * 16);
  run<0>(out, sms); run<1>(out, sms); run<2>(out, sms); run<3>(out, sms);
  run<6>(out, sms); run<7>(out, sms); run<9>(out, sms);
  return 0;
}
