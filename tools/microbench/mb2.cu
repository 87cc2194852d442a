// Step-0 micro-benchmark 2: does an SM gather from shared memory and from L2 at the same
// time faster than from either alone?  (Decides whether the config-4 kernel may split
// its gathers between the smem-resident tile and L2.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int NS, int NG>
__global__ void __launch_bounds__(512, 1) mixed(const uint4* __restrict__ g, uint32_t glines, uint4* out, int iters) {
  extern __shared__ uint4 sm[];
  const int rows = 1024;
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane8 = threadIdx.x & 7;
  uint32_t h = hash32(blockIdx.x * 4096 + (threadIdx.x >> 3));
  uint32_t h2 = hash32(h);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      h = h * 1664525u + 1013904223u;
      uint4 v = sm[((h >> 8) & (rows - 1)) * 8 + lane8];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      h2 = h2 * 1664525u + 1013904223u;
      uint4 v = __ldg(&g[(size_t)((h2 >> 4) & (glines - 1)) * 8 + lane8]);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int NS, int NG>
void run(const uint4* g, uint4* out, int sms) {
  cudaFuncSetAttribute(mixed<NS, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    mixed<NS, NG><<<sms, 512, 131072>>>(g, (32u << 20) / 128, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bs = (double)sms * 64 * iters * NS * 128, bg = (double)sms * 64 * iters * NG * 128;
    printf("{\"test\":\"mixed\",\"NS\":%d,\"NG\":%d,\"ms\":%.4f,\"smem_TBps\":%.2f,\"l2_TBps\":%.2f,\"total_TBps\":%.2f,\"B_clk_sm\":%.1f}\n",
           NS, NG, ms, bs / ms / 1e9, bg / ms / 1e9, (bs + bg) / ms / 1e9, (bs + bg) / (ms * 1e-3) / sms / 1.965e9);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* g; cudaMalloc(&g, 32 << 20); cudaMemset(g, 3, 32 << 20);
  uint4* out; cudaMalloc(&out, (size_t)sms * 512 * 16);
  run<8, 0>(g, out, sms); run<0, 8>(g, out, sms); run<6, 2>(g, out, sms); run<5, 3>(g, out, sms);
  run<4, 4>(g, out, sms); run<7, 1>(g, out, sms);
  cudaError_t e = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
