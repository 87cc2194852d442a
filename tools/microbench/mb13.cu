// Shared-memory cost of 64-B row gathers when half-groups of one warp read the SAME row in a step
// (a schedule-level "broadcast" reuse question: does a duplicated row cost fewer LSU wavefronts?).
// Each warp step: half-group h (lanes 4h..4h+3, 16 B per lane) reads 64-B tile row r_h.
// Row patterns per step (A..H = distinct random rows; "e"/"o" = forced even/odd parity):
//   0: Ae Bo Ce Do Ee Fo Ge Ho    8 distinct, parity-paired per phase (the SMEM kernel's rule)
//   1: Ae Ae Bo Bo Ce Ce Do Do    phase duplicates, phases alternate parity
//   2: A  A  B  B  C  C  D  D     phase duplicates, random parity
//   3: A  A  A  A  A  A  A  A     one row for the whole warp
//   4: Ae Ae Ce Do Ee Fo Ge Ho    one duplicated phase, the rest parity-paired
//   5: Ae Bo Ae Bo Ce Do Ce Do    duplicates across phases (phase 0 == phase 1, 2 == 3)
//   6: Ae Bo Ce Do Ae Bo Ce Do    duplicates across phases (phase 0 == 2, 1 == 3)
//   7: Ae Bo Ae Bo Ae Bo Ae Bo    two rows for the whole warp
//   8: Ae Ae Bo Bo Ce Do Ee Fo    two duplicated phases (even + odd row), two distinct pairs
//   9: Ae Be Ce De Ee Fe Ge He    8 distinct rows, all even (2-way conflict in every phase)
//  10: r, r+2, ..., r+14          8 distinct even rows of one 1-KB block
// Prints ns and clk per warp-LDS.128 for each pattern.  Result (profiles/r02_final/mb13_dup_rows_ncu.txt,
// ncu): every pattern 0-8 costs 4.0 shared wavefronts per LDS.128 -- rows shared by several
// half-groups of a step are NOT cheaper -- and 9/10 (same-parity rows) 8.0.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int PAT>
__global__ void __launch_bounds__(768, 1) gather_dup(uint4 *out, int rows, int iters) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < rows * 4; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 7, i * 11);
  __syncthreads();
  const int lane = threadIdx.x & 31, lane4 = lane & 3, hg = lane >> 2;
  const int warp = threadIdx.x >> 5;
  uint32_t s = hash32(blockIdx.x * 64 + warp);  // warp-uniform stream
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint32_t m = rows - 1;
  // 16 steps of addresses precomputed in registers, then replayed (the loop is LDS + XOR only)
  uint32_t addr[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    s = s * 1664525u + 1013904223u;
    const uint32_t h1 = hash32(s), h2 = hash32(s ^ 0x9e3779b9u);
    uint32_t cand[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) cand[j] = ((j < 4 ? h1 : h2) >> (8 * (j & 3))) * 2654435761u >> 21;
    uint32_t r;
    const uint32_t E = ~1u;
    if (PAT == 0) r = (hg & 1) ? (cand[hg] | 1) : (cand[hg] & E);
    else if (PAT == 1) r = ((hg >> 1) & 1) ? (cand[hg >> 1] | 1) : (cand[hg >> 1] & E);
    else if (PAT == 2) r = cand[hg >> 1];
    else if (PAT == 3) r = cand[0];
    else if (PAT == 4) r = hg < 2 ? (cand[0] & E) : ((hg & 1) ? (cand[hg] | 1) : (cand[hg] & E));
    else if (PAT == 5) { const int k = (hg & 1) + 2 * (hg >> 2); r = (hg & 1) ? (cand[k] | 1) : (cand[k] & E); }
    else if (PAT == 6) { const int k = hg & 3; r = (hg & 1) ? (cand[k] | 1) : (cand[k] & E); }
    else if (PAT == 7) r = (hg & 1) ? (cand[1] | 1) : (cand[0] & E);
    else if (PAT == 9) r = cand[hg] & E;
    else if (PAT == 10) r = (cand[0] & ~15u) + 2 * hg;
    else {
      if (hg < 4) r = (hg >> 1) ? (cand[1] | 1) : (cand[0] & E);
      else r = (hg & 1) ? (cand[hg] | 1) : (cand[hg] & E);
    }
    r &= m;
    addr[u] = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (r * 4 + lane4) * 16;
  }
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // rows move by 2 (same parity, same duplicates) on odd iterations: without it the compiler
    // merges the loads of two unrolled iterations (the first ncu run counted 8 LDS per iteration)
    const uint32_t odd = (it & 1) * 128;
#pragma unroll
    for (int u = 0; u < 16; u += 4) {
      uint4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w) : "r"(addr[u + q] + odd));
#pragma unroll
      for (int q = 0; q < 4; ++q) { acc.x ^= v[q].x; acc.y ^= v[q].y; acc.z ^= v[q].z; acc.w ^= v[q].w; }
    }
  }
  const long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0].x = static_cast<uint32_t>(c1 - c0);
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PAT>
void run(uint4 *out, int sms, int threads) {
  const int rows = 2048, iters = 2048;
  const size_t smem = rows * 64;
  cudaFuncSetAttribute(gather_dup<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gather_dup<PAT><<<sms, threads, smem>>>(out, rows, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  gather_dup<PAT><<<sms, threads, smem>>>(out, rows, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  uint32_t cyc = 0; cudaMemcpy(&cyc, out, 4, cudaMemcpyDeviceToHost);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double lds_per_sm = (double)(threads / 32) * iters * 16;
  printf("{\"pattern\":%d,\"threads\":%d,\"ms\":%.4f,\"clk_per_warp_lds\":%.3f,\"sm_cycles_per_warp_lds\":%.3f}\n", PAT,
         threads, ms, ms * 1e-3 * clk * 1e3 / lds_per_sm, cyc / lds_per_sm);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4 *out; cudaMalloc(&out, sms * 1024 * 16);
  for (int rep = 0; rep < 2; ++rep)
    for (int th : {512, 768}) {
      run<0>(out, sms, th); run<1>(out, sms, th); run<2>(out, sms, th); run<3>(out, sms, th);
      run<4>(out, sms, th); run<5>(out, sms, th); run<6>(out, sms, th); run<7>(out, sms, th);
      run<8>(out, sms, th); run<9>(out, sms, th); run<10>(out, sms, th);
    }
  return 0;
}
