// What does a schedule read cost next to the parity-paired 64-B gathers?  Every variant runs the
// gathers of mb8 variant 0 and adds, per 8 gathers, one read of 16 B of "schedule" per lane in a
// different access pattern:
//   0: nothing (baseline)
//   1: LDS.128, 8 distinct 16-B addresses in one 128-B line, 4 lanes each (today's chunk read)
//   2: LDS.128, every lane the same 16 B (warp-uniform)
//   3: LDS.32, 32 distinct 4-B words of one 128-B line (then 4 x SHFL within the half-group to
//      rebuild the 16-B chunk)
//   4: LDC (constant cache), warp-uniform 16 B
//   5: LDC, 8 distinct 16-B addresses (4 lanes each)
//   6: LDG.128 through L1 (ld.global.nc), 8 distinct 16-B addresses, L1-resident table
// Prints clk per warp-gather per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ uint4 c_tab[2048];

template <int V>
__global__ void __launch_bounds__(512, 1) mix(uint4 *out, const uint4 *__restrict__ gtab, int rows, int iters) {
  extern __shared__ __align__(128) uint4 sm[];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < rows * 4 + 2048; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const uint4 *tab = sm + rows * 4;  // 32 KB "schedule" after the tile
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1, hg = lane >> 2;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  uint4 acc = make_uint4(0, 0, 0, 0);
  uint32_t sacc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
      uint32_t r = half ? (rb | 1) : (ra & ~1u);
      uint4 v = sm[r * 4 + lane4];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    const uint32_t line = ((it * 24 + warp) * 8) & 2047;  // 128-B line of the table (8 uint4)
    if (V == 1) { uint4 s = tab[(line & ~7u) + hg]; sacc ^= s.x ^ s.y ^ s.z ^ s.w; }
    if (V == 2) { uint4 s = tab[line]; sacc ^= s.x ^ s.y ^ s.z ^ s.w; }
    if (V == 3) {
      uint32_t w = reinterpret_cast<const uint32_t *>(tab + (line & ~7u))[lane];
      uint32_t a0 = __shfl_sync(0xffffffffu, w, (lane & ~3) | 0), a1 = __shfl_sync(0xffffffffu, w, (lane & ~3) | 1);
      uint32_t a2 = __shfl_sync(0xffffffffu, w, (lane & ~3) | 2), a3 = __shfl_sync(0xffffffffu, w, (lane & ~3) | 3);
      sacc ^= a0 ^ a1 ^ a2 ^ a3;
    }
    if (V == 4) { uint4 s = c_tab[line]; sacc ^= s.x ^ s.y ^ s.z ^ s.w; }
    if (V == 5) { uint4 s = c_tab[(line & ~7u) + hg]; sacc ^= s.x ^ s.y ^ s.z ^ s.w; }
    if (V == 6) { uint4 s = __ldg(gtab + (line & ~7u) + hg); sacc ^= s.x ^ s.y ^ s.z ^ s.w; }
    acc.x ^= sacc;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(uint4 *out, const uint4 *gtab, int sms) {
  const int rows = 2048, iters = 2048, threads = 512;
  const size_t smem = rows * 64 + 2048 * 16;
  cudaFuncSetAttribute(mix<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mix<V><<<sms, threads, smem>>>(out, gtab, rows, 8);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("variant %d: %s\n", V, cudaGetErrorString(e)); return; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    mix<V><<<sms, threads, smem>>>(out, gtab, rows, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double gathers = (double)sms * (threads / 32) * iters * 8;
  printf("{\"variant\":%d,\"ms\":%.4f,\"clk_per_gather_per_sm\":%.3f}\n", V, best,
         best * 1e-3 * clk * 1e3 / (gathers / sms));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4 *out, *gtab;
  cudaMalloc(&out, 1024 * 512 * 16);
  cudaMalloc(&gtab, 2048 * 16);
  cudaMemset(gtab, 1, 2048 * 16);
  uint4 host[2048];
  for (int i = 0; i < 2048; ++i) host[i] = make_uint4(i, i + 1, i + 2, i + 3);
  cudaMemcpyToSymbol(c_tab, host, sizeof(host));
  run<0>(out, gtab, sms); run<1>(out, gtab, sms); run<2>(out, gtab, sms); run<3>(out, gtab, sms);
  run<4>(out, gtab, sms); run<5>(out, gtab, sms); run<6>(out, gtab, sms);
  return 0;
}
