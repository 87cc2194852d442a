// Store-path cost inside an L2 gather stream (config 5's band kernel: one 512-B coded-row store
// per ~6 gathers).  Each warp gathers B=4 random 512-B rows (16 B per lane) from a 25.9 MB
// L2-resident band (50,500 rows at an 8-KB stride), XORs, and every `every` batches stores its
// accumulator as one 512-B row by store variant V:
//   0 none, 1 st.global.cs, 2 st.global (write-back), 3 st.global.L1::no_allocate,
//   4 st.global.L2::cache_hint evict_first, 5 TMA bulk store (STS to a per-warp smem slot,
//   fence.proxy.async, cp.async.bulk.global.shared::cta by lane 0), 6 st.global.v8 (lanes 0-15
//   store 32 B each after a shuffle: 16 lanes per 512 B)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb11 mb11.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int V>
__global__ void __launch_bounds__(256) k(const uint8_t *g, uint8_t *wr, uint4 *out, uint32_t iters, uint32_t every) {
  __shared__ __align__(128) uint4 slot[8][32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t h = hash32(blockIdx.x * 1024 + w + 777);
  uint4 acc = make_uint4(0, 0, 0, 0);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint64_t wrow = (static_cast<uint64_t>(blockIdx.x) * 8 + w) * 977;
  for (uint32_t it = 0; it < iters; ++it) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      h = h * 1664525u + 1013904223u;
      const uint32_t r = (h >> 7) % 50500u;
      const uint8_t *p = g + static_cast<uint64_t>(r) * 8192 + lane * 16;
      asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    if (V != 0 && (it % every) == every - 1) {
      wrow = (wrow + 7919) % 60000ull;
      uint8_t *dst = wr + wrow * 8192 + (h & 15) * 512;
      if (V == 1) __stcs(reinterpret_cast<uint4 *>(dst + lane * 16), acc);
      if (V == 2) *reinterpret_cast<uint4 *>(dst + lane * 16) = acc;
      if (V == 3) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" :: "l"(dst + lane * 16), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
      if (V == 4) asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" :: "l"(dst + lane * 16), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w), "l"(pol) : "memory");
      if (V == 5) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot free again
        __syncwarp();
        slot[w][lane] = acc;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" :: "l"(dst),
                       "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&slot[w][0]))) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (V == 6) {
        uint4 o;  // lane l < 16 stores bytes [32l, 32l+32) = lanes 2l and 2l+1
        o.x = __shfl_sync(0xffffffffu, acc.x, (2 * lane + 1) & 31);
        o.y = __shfl_sync(0xffffffffu, acc.y, (2 * lane + 1) & 31);
        o.z = __shfl_sync(0xffffffffu, acc.z, (2 * lane + 1) & 31);
        o.w = __shfl_sync(0xffffffffu, acc.w, (2 * lane + 1) & 31);
        uint4 a2;
        a2.x = __shfl_sync(0xffffffffu, acc.x, (2 * lane) & 31);
        a2.y = __shfl_sync(0xffffffffu, acc.y, (2 * lane) & 31);
        a2.z = __shfl_sync(0xffffffffu, acc.z, (2 * lane) & 31);
        a2.w = __shfl_sync(0xffffffffu, acc.w, (2 * lane) & 31);
        if (lane < 16)
          asm volatile("st.global.cs.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" :: "l"(dst + lane * 32), "r"(a2.x), "r"(a2.y), "r"(a2.z), "r"(a2.w), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
      }
      acc = make_uint4(0, 0, 0, 0);
    }
  }
  if (V == 5 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(const uint8_t *g, uint8_t *wr, uint4 *out, int blocks_per_sm, uint32_t every) {
  const int blocks = 148 * blocks_per_sm;
  const uint32_t iters = 1024;
  k<V><<<blocks, 256>>>(g, wr, out, 16, every);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<V><<<blocks, 256>>>(g, wr, out, iters, every);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double gb = (double)blocks * 8 * iters * 4 * 512;
  printf("V%d warps/SM %2d store every %u batches: %.3f ms  gathers %.2f TB/s  %s\n", V, blocks_per_sm * 8, every, ms,
         gb / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  uint8_t *g = nullptr, *wr = nullptr; uint4 *out = nullptr;
  if (cudaMalloc(&g, 50500ull * 8192) || cudaMalloc(&wr, 60000ull * 8192) || cudaMalloc(&out, 148ull * 8 * 256 * 16)) return 1;
  cudaMemset(g, 1, 50500ull * 8192);
  for (int bps : {4, 6}) {
    run<0>(g, wr, out, bps, 2);
    run<1>(g, wr, out, bps, 2);
    run<2>(g, wr, out, bps, 2);
    run<3>(g, wr, out, bps, 2);
    run<4>(g, wr, out, bps, 2);
    run<5>(g, wr, out, bps, 2);
    run<6>(g, wr, out, bps, 2);
  }
  return 0;
}
