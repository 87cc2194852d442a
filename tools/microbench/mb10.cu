// L2 random-gather rate vs the address stride of the gathered rows (config 5's band layout).
// Each warp gathers B rows at a time (16 B per lane = 512 B per row, as fsb_lt_band) from
// `rows` rows spaced `stride` bytes apart (stride 512: a contiguous block, as tools/microbench/
// mb7.cu PAT 3; stride 8192: one 512-B band of every 8-KB symbol, config 5), XORs them, repeat.
// Prints TB/s of gathered bytes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mb10.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int B>
__global__ void gather(const uint8_t *g, uint4 *out, uint32_t rows, uint32_t stride, uint32_t iters, uint8_t *wr = nullptr,
                       uint32_t wr_every = 0) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t h = hash32(blockIdx.x * 1024 + (threadIdx.x >> 5) + 12345);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint32_t it = 0; it < iters; ++it) {
    uint4 v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      h = h * 1664525u + 1013904223u;
      const uint32_t r = (h >> 7) % rows;
      const uint8_t *p = g + static_cast<uint64_t>(r) * stride + lane * 16;
      asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < B; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    if (wr_every && (it % wr_every) == 0) {  // a streaming 512-B row store (as a coded row of fsb_lt_band)
      const uint64_t w = (static_cast<uint64_t>(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * iters + it) % 60000ull;
      __stcs(reinterpret_cast<uint4 *>(wr + w * 8192 + (h & 15) * 512 + lane * 16), acc);
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int B>
void run(const uint8_t *g, uint4 *out, uint32_t rows, uint32_t stride, int warps_per_sm, const char *tag, uint8_t *wr = nullptr,
         uint32_t every = 0) {
  const int threads = 256, sms = 148;
  const int blocks = sms * warps_per_sm / 8;
  const uint32_t iters = 4096 / B;
  gather<B><<<blocks, threads>>>(g, out, rows, stride, 16, wr, every);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  gather<B><<<blocks, threads>>>(g, out, rows, stride, iters, wr, every);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)blocks * threads / 32 * iters * B * 512;
  fflush(stdout);
  printf("%-28s rows %6u stride %5u warps/SM %2d B %d: %.3f ms %.2f TB/s %s\n", tag, rows, stride, warps_per_sm, B, ms,
         bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint8_t *g = nullptr; uint4 *out = nullptr;
  const size_t bytes = 50500ull * 8704 + 65536;
  cudaError_t e1 = cudaMalloc(&g, bytes), e2 = cudaMalloc(&out, 148ull * 64 * 256 * 16);
  printf("malloc: %s %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
  fflush(stdout);
  if (e1 != cudaSuccess || e2 != cudaSuccess) return 1;
  cudaMemset(g, 1, bytes);
  // working-set sweep: random 512-B rows of `rows` rows at a 512-B stride (a contiguous region)
  for (uint32_t mb : {8u, 16u, 26u, 40u, 52u, 64u, 80u, 100u, 128u, 200u, 400u}) {
    char tag[64];
    snprintf(tag, sizeof(tag), "contig %u MB", mb);
    run<4>(g, out, mb * 2048u, 512, 48, tag);
  }
  for (uint32_t mb : {26u, 52u, 78u}) {
    char tag[64];
    snprintf(tag, sizeof(tag), "8K-stride bands %u MB", mb);
    run<4>(g, out, mb * 2048u / 16u * 16u, 8192 / (mb / 26u), 48, tag);
  }
  return 0;
}
