// Step-0 micro-benchmarks: device properties, shared-memory
// random-row gather bandwidth, L2 random-line gather bandwidth, HBM streaming
// bandwidth. Not part of the product; numbers feed DESIGN.md's rooflines.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// Each 8-lane group reads one random 128-B row of a smem buffer of `rows` rows per step.
__global__ void __launch_bounds__(512, 1) smem_gather(uint4* out, int rows, int iters) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane8 = threadIdx.x & 7;
  const int grp = threadIdx.x >> 3;
  uint32_t h = hash32(blockIdx.x * 4096 + grp);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t r = (h >> 8) & (rows - 1);
      uint4 v = sm[r * 8 + lane8];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Each 8-lane group reads one random 128-B line of a global buffer per step.
__global__ void l2_gather(const uint4* __restrict__ src, uint4* out, uint32_t lines, int iters) {
  const int lane8 = threadIdx.x & 7;
  uint32_t h = hash32(blockIdx.x * 1024 + (threadIdx.x >> 3));
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t r = (h >> 4) & (lines - 1);
      uint4 v = __ldg(&src[(size_t)r * 8 + lane8]);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void stream_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

__global__ void clk_kernel(long long* out) {
  long long t0 = clock64();
  while (clock64() - t0 < 200000000LL) {}
  out[0] = clock64() - t0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int l2win = 0, persist = 0, optin = 0, clk = 0;
  cudaDeviceGetAttribute(&l2win, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"persist_max\":%d,\"window_max\":%d,"
         "\"smem_optin\":%d,\"smem_per_sm\":%zu,\"clock_khz\":%d,\"cc\":\"%d.%d\"}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, persist, l2win, optin,
         p.sharedMemPerMultiprocessor, clk, p.major, p.minor);
  const int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint4* out; CK(cudaMalloc(&out, (size_t)sms * 4 * 1024 * 16));

  // smem gather: 1040 rows x 128 B = 133 KB, 512 threads, 1 CTA/SM
  {
    int rows = 1024; size_t smem = (size_t)rows * 128;
    CK(cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int iters = 4000;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      smem_gather<<<sms, 512, smem>>>(out, rows, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)sms * 64 /*groups*/ * iters * 8 * 128;
      printf("{\"test\":\"smem_gather\",\"rows\":%d,\"ms\":%.4f,\"TBps\":%.3f,\"B_per_clk_sm_at_1965\":%.2f}\n",
             rows, ms, bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  // L2 gather from 16/32/64 MB, and 1 GB (HBM)
  {
    size_t maxb = (size_t)1 << 30; uint4* src; CK(cudaMalloc(&src, maxb));
    CK(cudaMemset(src, 1, maxb));
    size_t sizes[4] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20, maxb};
    for (int s = 0; s < 4; ++s) {
      uint32_t lines = (uint32_t)(sizes[s] / 128);
      int iters = 200; int blocks = sms * 8;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        l2_gather<<<blocks, 256>>>(src, out, lines, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double bytes = (double)blocks * 32 * iters * 8 * 128;
        printf("{\"test\":\"global_gather\",\"MB\":%zu,\"ms\":%.4f,\"TBps\":%.3f}\n", sizes[s] >> 20, ms,
               bytes / ms / 1e9);
      }
    }
    uint4* dst; CK(cudaMalloc(&dst, maxb));
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      stream_copy<<<sms * 8, 512>>>(src, dst, maxb / 16);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"test\":\"stream_copy\",\"GB\":1.07,\"ms\":%.4f,\"GBps_rw\":%.1f}\n", ms, 2.0 * maxb / ms / 1e6);
    }
    cudaFree(src); cudaFree(dst);
  }
  {
    long long* d; cudaMalloc(&d, 8);
    cudaEventRecord(e0); clk_kernel<<<1, 1>>>(d); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"test\":\"sm_clock\",\"MHz\":%.1f}\n", c / (ms * 1e3));
  }
  return 0;
}
