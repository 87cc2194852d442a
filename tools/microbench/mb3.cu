// Shared-memory bank behaviour of 64-B row gathers (the SMEM kernel's access pattern).
// Each warp: lanes 8q..8q+3 (half 0) read 64 B of row a, lanes 8q+4..8q+7 (half 1) 64 B of row b,
// with 16 B per lane.  Patterns (per step, per group):
//   0: a even, b odd (the host schedule's bank rule)
//   1: a, b both even
//   2: a, b random
//   4: schedule-chunk load: half-group h (4 lanes) reads 16-B word h of a 128-B chunk
//   5: contiguous 512-B load (lane l reads 16-B word l)
// Prints ns and smem bytes/clk/SM for each pattern.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int PAT>
__global__ void __launch_bounds__(512, 1) gather64(uint4* out, int rows, int iters) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1;
  const int grp = threadIdx.x >> 3;
  uint32_t h = hash32(blockIdx.x * 4096 + grp);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
      uint32_t r, idx;
      if (PAT == 0) r = half ? (rb | 1) : (ra & ~1u);
      else if (PAT == 1) r = half ? (rb & ~1u) : (ra & ~1u);
      else r = half ? rb : ra;
      idx = r * 4 + lane4;
      if (PAT == 4) idx = (ra & ~7u) + (lane >> 2);
      if (PAT == 5) idx = ((ra & ~31u) + lane) & (rows * 4 - 1);
      uint4 v = sm[idx];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PAT>
void run(uint4* out, int sms) {
  const int rows = 2048, iters = 4096, threads = 512;
  const size_t smem = rows * 64;
  cudaFuncSetAttribute(gather64<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gather64<PAT><<<sms, threads, smem>>>(out, rows, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  gather64<PAT><<<sms, threads, smem>>>(out, rows, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = (double)sms * threads * iters * 8 * 16;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"pattern\":%d,\"ms\":%.4f,\"TBps\":%.3f,\"B_per_clk_sm\":%.2f}\n", PAT, ms, bytes / ms / 1e9,
         bytes / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out; cudaMalloc(&out, sms * 512 * 16);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>(out, sms); run<1>(out, sms); run<2>(out, sms); run<4>(out, sms); run<5>(out, sms);
  }
  return 0;
}
