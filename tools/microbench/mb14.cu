// Tensor memory (TMEM) as a gather source: how fast can warps read arbitrary TMEM columns?
// Candidate design: source rows of a tile live in TMEM (columns = rows, lanes = byte offsets), a
// warp gathers one source per tcgen05.ld at a warp-uniform column, so the gathers do not touch the
// shared-memory (L1TEX LSU) port at all.  Each warp reads its own lane quarter (32 * (warp % 4)).
//   variant  N   batch  what
//   1        x1  8      tcgen05.ld.32x32b.x1 at pseudo-random columns, wait::ld per batch, XOR
//   2        x1  16
//   3        x1  32
//   4        x2  8      2 consecutive columns per load (8 B per lane)
//   5        x4  8      4 consecutive columns per load (16 B per lane)
//   6        x4  16
//   7        x1  16 + 8 parity-paired 64-B shared-memory LDS.128 gathers per batch (both pipes)
//   8        smem only: 8 LDS.128 gathers per batch (mb8 variant 0 reference)
// Prints bytes per clock per SM delivered into registers by TMEM (and by shared memory).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int N>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t* v) {
  if constexpr (N == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(taddr) : "memory");
  } else if constexpr (N == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(taddr) : "memory");
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr)
                 : "memory");
  }
}

template <int V, int N, int B>
__global__ void __launch_bounds__(1024, 1) tg(uint32_t* out, int iters) {
  extern __shared__ __align__(128) uint4 sm[];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const int rows = 1024;
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  // fill this warp's quarter (every warp of a quarter writes all 512 columns: harmless duplicates)
  if (warp < 4) {
    for (int c = 0; c < 512; c += 4) {
      const uint32_t a = tbase + ((32u * (warp & 3)) << 16) + c;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(c * 131 + lane),
                   "r"(c * 7 + lane), "r"(c ^ lane), "r"(c + 3 * lane)
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t qbase = tbase + ((32u * (warp & 3)) << 16);
  uint32_t hw = (blockIdx.x * 4096 + warp) * 2654435761u;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  const int lane4 = lane & 3, half = (lane >> 2) & 1;
  uint32_t acc = 0;
  uint4 sacc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    if (V != 8) {
      uint32_t v[B][N];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        hw = hw * 1664525u + 1013904223u;
        const uint32_t col = (hw >> 20) & (511u & ~(uint32_t)(N - 1));
        tm_ld<N>(qbase + col, v[u]);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < B; ++u)
#pragma unroll
        for (int e = 0; e < N; ++e) acc ^= v[u][e];
    }
    if (V == 7 || V == 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        h = h * 1664525u + 1013904223u;
        uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
        uint32_t r = half ? (rb | 1) : (ra & ~1u);
        uint4 x = sm[r * 4 + lane4];
        sacc.x ^= x.x; sacc.y ^= x.y; sacc.z ^= x.z; sacc.w ^= x.w;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  if ((acc ^ sacc.x ^ sacc.y ^ sacc.z ^ sacc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int N, int B>
void run(uint32_t* out, int sms, int threads) {
  const int iters = 4096;
  const size_t smem = 1024 * 64 + 100 * 1024;  // one CTA per SM
  cudaFuncSetAttribute(tg<V, N, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tg<V, N, B><<<sms, threads, smem>>>(out, 8);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("variant %d: %s\n", V, cudaGetErrorString(e)); return; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  tg<V, N, B><<<sms, threads, smem>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double warps = threads / 32;
  const double tm_bytes = (V == 8) ? 0 : warps * iters * B * N * 128.0;
  const double sm_bytes = (V == 7 || V == 8) ? warps * iters * 8 * 512.0 : 0;
  printf("{\"variant\":%d,\"x\":%d,\"batch\":%d,\"warps\":%d,\"ms\":%.4f,\"tmem_B_per_clk_sm\":%.1f,"
         "\"smem_B_per_clk_sm\":%.1f,\"clk_per_tmem_ld_per_quarter\":%.3f}\n",
         V, N, B, threads / 32, ms, tm_bytes / cycles, sm_bytes / cycles,
         (V == 8) ? 0.0 : cycles / (warps * iters * B / 4.0));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 1024 * 1024 * 4);
  for (int threads : {128, 256, 512, 1024}) {
    run<1, 1, 8>(out, sms, threads);
    run<2, 1, 16>(out, sms, threads);
    run<3, 1, 32>(out, sms, threads);
    run<4, 2, 8>(out, sms, threads);
    run<5, 4, 8>(out, sms, threads);
    run<6, 4, 16>(out, sms, threads);
    run<7, 1, 16>(out, sms, threads);
    run<8, 1, 8>(out, sms, threads);
  }
  return 0;
}
