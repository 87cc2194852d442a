// Does the shared-memory bank of a 64-B row depend only on address bit 6?  Parity-paired
// 64-B row gathers (half 0 even row, half 1 odd row) from a 4096-row window placed at a
// byte offset OFF of a 227 KB dynamic allocation, plus "mixed": half 0 in the low window,
// half 1 in the high window.  Prints bytes/clk/SM and is meant to run under ncu for the
// bank-conflict counter.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) g64(uint4* out, uint32_t off_a, uint32_t off_b, int rows, int iters) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < 232448 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (half ? off_b : off_a) + lane4 * 16;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t r = ((h >> 8) % rows);
      r = half ? (r | 1) : (r & ~1u);
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(base + r * 64));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out; cudaMalloc(&out, sms * 512 * 16);
  const int smem = 232448;
  cudaFuncSetAttribute(g64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct { uint32_t a, b; int rows; const char* name; } cases[] = {
      {0, 0, 1024, "low64K"}, {65536, 65536, 1024, "64K-128K"}, {131072, 131072, 1024, "128K-192K"},
      {163840, 163840, 1024, "160K-224K"}, {0, 131072, 1024, "mixed_low_high"}, {0, 0, 3600, "0-225K"},
      {86016, 86016, 1024, "84K-148K"}};
  for (auto& c : cases) {
    const int iters = 2048;
    g64<<<sms, 512, smem>>>(out, c.a, c.b, c.rows, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    g64<<<sms, 512, smem>>>(out, c.a, c.b, c.rows, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)sms * 512 * iters * 8 * 16;
    printf("{\"case\":\"%s\",\"ms\":%.4f,\"B_per_clk_sm\":%.2f}\n", c.name, ms, bytes / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
