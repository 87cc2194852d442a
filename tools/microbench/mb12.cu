// TMEM read throughput for gathers: warps of each lane quarter issue tcgen05.ld.32x32b.x{1,2,4}
// at pseudo-random (warp-uniform) column addresses, N loads then one tcgen05.wait::ld, XOR into a
// register.  Prints bytes/clk/SM of TMEM -> register traffic, next to an ld.shared gather loop of
// the same shape (one 128-B row per warp instruction, 4 B per lane) for comparison.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb12 mb12.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int X, int N, bool kShared>
__global__ void __launch_bounds__(1024, 1) k(uint32_t *out, uint32_t iters) {
  __shared__ uint32_t taddr_s;
  __shared__ __align__(128) uint32_t sm[256 * 32];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t i = threadIdx.x; i < 256 * 32; i += blockDim.x) sm[i] = i * 2654435761u;
  if (!kShared && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&taddr_s))) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = kShared ? 0 : taddr_s + ((32u * (warp & 3)) << 16);
  uint32_t h = 0x9E3779B9u * (warp + 1 + blockIdx.x * 64);
  uint32_t acc = 0;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + lane * 4;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t v[N * X];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      h = h * 1664525u + 1013904223u;
      const uint32_t col = (h >> 20) & (512 - X);  // warp-uniform
      if (kShared) {
#pragma unroll
        for (int x = 0; x < X; ++x)
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[u * X + x]) : "r"(sbase + ((col + x) & 255) * 128));
      } else if (X == 1) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[u]) : "r"(tbase + col));
      } else if (X == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v[2 * u]), "=r"(v[2 * u + 1]) : "r"(tbase + col));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[4 * u]), "=r"(v[4 * u + 1]), "=r"(v[4 * u + 2]), "=r"(v[4 * u + 3]) : "r"(tbase + col));
      }
    }
    if (!kShared) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < N * X; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (!kShared && warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s) : "memory");
}

template <int X, int N, bool kShared>
void run(uint32_t *out, int warps) {
  const uint32_t iters = 4096;
  k<X, N, kShared><<<148, warps * 32>>>(out, 8);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<X, N, kShared><<<148, warps * 32>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bytes = 148.0 * warps * iters * N * X * 128;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%s x%d N%d warps %2d: %.3f ms  %.1f B/clk/SM  %s\n", kShared ? "ld.shared " : "tcgen05.ld", X, N, warps, ms,
         bytes / cyc / 148, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  uint32_t *out;
  cudaMalloc(&out, 148 * 1024 * 4);
  for (int w : {8, 16, 32}) {
    run<1, 8, false>(out, w);
    run<2, 4, false>(out, w);
    run<4, 2, false>(out, w);
    run<1, 16, false>(out, w);
    run<1, 8, true>(out, w);
  }
  return 0;
}
