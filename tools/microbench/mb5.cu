// Which shared-memory op mix produces the bank-conflict counts seen in fsb_smem_encode?
// Every variant does parity-paired 64-B row gathers (conflict-free, measured in mb3.cu) and adds
// one op per 8 gathers: 1 schedule-chunk load (half-group h reads 16-B word h of a 128-B chunk),
// 2 warp shuffles (xor 4), 3 a 16-B global store per lane, 4 all lanes gather the same 2 rows,
// 5 gathers where the 4 groups read the same even/odd row pair (cross-phase duplicates),
// 6 a 16-B global store per lane where each half-group (4 lanes, 64 B) writes its own 4-KB-strided
//   row (8 distinct 128-B lines per store, the SMEM kernel's coded-row store),
// 7 as 6 but each group (8 lanes, 128 B) writes one full line (4 lines per store),
// 8 as 6 but staged: each half-group writes its 64 B to a per-warp shared staging slot (STS) and
//   lane 4h issues a 64-B cp.async.bulk shared->global copy of it (double-buffered staging).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(512, 1) mix(uint4* out, int rows, int iters) {
  extern __shared__ uint4 sm[];
  __shared__ __align__(128) uint4 stage[16][2][32];  // warp, buffer, 8 half-groups x 4 lanes
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, half = (lane >> 2) & 1;
  uint32_t h = (blockIdx.x * 4096 + (threadIdx.x >> 3)) * 2654435761u;
  uint32_t hw = (blockIdx.x * 4096 + (threadIdx.x >> 5)) * 2654435761u;  // warp-uniform
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      hw = hw * 1664525u + 1013904223u;
      uint32_t ra = (h >> 8) & (rows - 1), rb = (h >> 20) & (rows - 1);
      if (V == 5) { ra = (hw >> 8) & (rows - 1); rb = (hw >> 20) & (rows - 1); }
      uint32_t r = half ? (rb | 1) : (ra & ~1u);
      if (V == 4) r = half;
      uint4 v = sm[r * 4 + lane4];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if (V == 1) {
      uint4 v = sm[((hw >> 8) & (rows - 1) & ~7u) + (lane >> 2)];
      acc.x += v.x;
    }
    if (V == 2) {
      acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, 4);
      acc.z ^= __shfl_xor_sync(0xffffffffu, acc.z, 4);
    }
    if (V == 3) out[(blockIdx.x * blockDim.x + threadIdx.x + it * 64) & (1024 * 512 - 1)] = acc;
    if (V == 6) {
      const uint32_t row = (hw + (threadIdx.x >> 2) * 7919u) & 2047u;  // 2048 rows of 4 KB
      out[(row * 256 + blockIdx.x * 4 + lane4) & (1024 * 512 - 1)] = acc;
    }
    if (V == 8) {
      const uint32_t w = threadIdx.x >> 5, buf = it & 1;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer `buf` reusable
      __syncwarp();
      stage[w][buf][lane] = acc;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane4 == 0) {
        const uint32_t row = (hw + (threadIdx.x >> 2) * 7919u) & 2047u;
        uint4* dst = out + ((row * 256 + blockIdx.x * 4) & (1024 * 512 - 1));
        const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(&stage[w][buf][lane]));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(dst), "r"(src) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (V == 9 || V == 10 || V == 11) {  // as 6 with explicit cache operators
      const uint32_t row = (hw + (threadIdx.x >> 2) * 7919u) & 2047u;
      uint4* dst = out + ((row * 256 + blockIdx.x * 4 + lane4) & (1024 * 512 - 1));
      if (V == 9)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
      if (V == 10)
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
      if (V == 11)
        asm volatile("st.global.wt.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(acc.x), "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
    }
    if (V == 7) {
      const uint32_t row = (hw + (threadIdx.x >> 3) * 7919u) & 2047u;
      out[(row * 256 + blockIdx.x * 8 + (lane & 7)) & (1024 * 512 - 1)] = acc;
    }
  }
  if (V == 8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(uint4* out, int sms) {
  const int rows = 2048, iters = 2048, threads = 512;
  const size_t smem = rows * 64;
  cudaFuncSetAttribute(mix<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mix<V><<<sms, threads, smem>>>(out, rows, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  mix<V><<<sms, threads, smem>>>(out, rows, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double gathers = (double)sms * (threads / 32) * iters * 8;  // warp-level gather LDS
  printf("{\"variant\":%d,\"ms\":%.4f,\"clk_per_gather_per_sm\":%.3f}\n", V, ms,
         ms * 1e-3 * clk * 1e3 / (gathers / sms));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out; cudaMalloc(&out, 1024 * 512 * 16);
  run<0>(out, sms); run<1>(out, sms); run<2>(out, sms); run<3>(out, sms); run<5>(out, sms);
  run<6>(out, sms); run<7>(out, sms); run<8>(out, sms); run<9>(out, sms); run<10>(out, sms); run<11>(out, sms);
  return 0;
}
