// Distributed shared memory (DSMEM) gather bandwidth: can a thread-block cluster hold a tile too
// large for one SM (config 5: K x 64 B = 3.2 MB) and serve random 64-B row gathers fast enough?
// Each CTA of a cluster of C fills `rows` 64-B rows of its shared memory; every warp then
// gathers random 64-B rows (4 lanes x 16 B per row, 8 rows per warp instruction, parity-paired
// as in the SMEM kernel) from a random CTA of the cluster (PAT 1) or from its own CTA (PAT 0,
// through the shared::cluster window), or via plain ld.shared (PAT 2, reference).
// Also PAT 3: random rows from global memory (L2-resident 25.9 MB band), for the L2 rate.
// Prints bytes/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank)); return r;
}
__device__ __forceinline__ uint4 ld_cluster(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 ld_shared(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int PAT>
__global__ void __launch_bounds__(512, 1) dsm(uint4* out, const uint4* g, int rows, int grows, int csize, int iters) {
  extern __shared__ __align__(128) uint4 sm[];
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  cluster_sync();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1;
  const int grp = threadIdx.x >> 3;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  uint32_t bases[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bases[c] = PAT == 1 || PAT == 0 ? mapa(base, c < csize ? c : 0) : base;
  const uint32_t me = cluster_rank();
  uint32_t h = hash32(blockIdx.x * 4096 + grp);
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
      uint32_t r = half ? (rb | 1) : (ra & ~1u);
      if (PAT == 3) {
        uint32_t gr = (h >> 4) % grows;
        v[u] = __ldg(g + static_cast<size_t>(gr) * 32 + (lane & 31));  // 512-B row band, lane 16 B
      } else {
        uint32_t c = PAT == 1 ? (h >> 1) % csize : me;
        uint32_t b = bases[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) b = (c == q) ? bases[q] : b;
        uint32_t addr = b + (r * 4 + lane4) * 16;
        v[u] = PAT == 2 ? ld_shared(base + (r * 4 + lane4) * 16) : ld_cluster(addr);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  cluster_sync();
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PAT>
void run(uint4* out, const uint4* g, int csize, int grows) {
  const int rows = 2048, iters = 2048, threads = 512;
  const size_t smem = rows * 64;
  cudaFuncSetAttribute(dsm<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(dsm<PAT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int grid = (148 / csize) * csize;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dsm<PAT>, out, g, rows, grows, csize, 16);
  if (e != cudaSuccess) { printf("PAT %d csize %d: launch error %s\n", PAT, csize, cudaGetErrorString(e)); return; }
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, dsm<PAT>, out, g, rows, grows, csize, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  e = cudaGetLastError();
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = (double)grid * threads * iters * 8 * 16;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("PAT %d (%s) csize %2d grid %3d: %.3f ms  %.1f B/clk/SM  %.1f TB/s  %s\n", PAT,
         PAT == 0 ? "dsmem-own" : PAT == 1 ? "dsmem-rand" : PAT == 2 ? "ld.shared" : "L2-gather",
         csize, grid, ms, bytes / cyc / grid, bytes / (ms * 1e-3) / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  uint4* out; cudaMalloc(&out, 148 * 512 * 16);
  const int grows = 50500;                         // config 5 band: K rows x 512 B
  uint4* g; cudaMalloc(&g, (size_t)grows * 512);
  cudaMemset(g, 1, (size_t)grows * 512);
  run<2>(out, g, 1, grows);
  for (int c : {2, 4, 8, 16}) run<0>(out, g, c, grows);
  for (int c : {2, 4, 8, 16}) run<1>(out, g, c, grows);
  run<3>(out, g, 1, grows);
  return 0;
}
