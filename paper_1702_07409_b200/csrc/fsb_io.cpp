// Host-buffer encode (fs_encode_host): the library's staging pipeline between host memory and
// the encode kernels, so a caller with data in (pinned) host memory gets the copies in both
// directions overlapped with the kernels.  Work is split into chunks issued alternately on two
// library-owned streams:
//   - several stripes (stripes are independent): chunks of whole stripes, one
//     strided 2D copy per buffer and direction, fs_encode_stripes semantics per chunk;
//   - one stripe: chunks of byte columns (>= 2 KB; XOR is bytewise, so a column range of the
//     output depends only on the same columns of the input -- the fs_encode_range partition),
//     2D copies of the column block of every row.
// The staging buffers live with the graph (grown on demand, freed by fs_free).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "fsb_internal.h"

namespace fsb {

IoCache::~IoCache() {
  if (device < 0) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (int j = 0; j < 2; ++j) {
    if (st[j]) cudaStreamSynchronize(st[j]);
    if (done[j]) cudaEventDestroy(done[j]);
    if (st[j]) cudaStreamDestroy(st[j]);
  }
  if (start) cudaEventDestroy(start);
  if (buf) cudaFree(buf);
  if (prev >= 0) cudaSetDevice(prev);
}

static fs_status io_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FS_ECUDA;
}

fs_status encode_host(const Graph &g, IoCache &c, uint32_t S, const uint8_t *h_data, uint64_t data_stride,
                      uint8_t *h_checks, uint64_t checks_stride, uint8_t *h_coded, uint64_t coded_stride,
                      uint32_t chunks, void *stream_ptr, uint32_t *launches) {
  *launches = 0;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  cudaError_t e;
  if (c.device < 0) {
    c.device = g.dev.device;
    for (int j = 0; j < 2; ++j) {
      if ((e = cudaStreamCreateWithFlags(&c.st[j], cudaStreamNonBlocking)) != cudaSuccess)
        return io_fail(e, "cudaStreamCreateWithFlags");
      if ((e = cudaEventCreateWithFlags(&c.done[j], cudaEventDisableTiming)) != cudaSuccess)
        return io_fail(e, "cudaEventCreate");
    }
    if ((e = cudaEventCreateWithFlags(&c.start, cudaEventDisableTiming)) != cudaSuccess)
      return io_fail(e, "cudaEventCreate");
  }
  const uint64_t k = g.prm.k, p = g.prm.p, n = g.prm.n, t = g.prm.t;
  const uint64_t rows = k + p + n;
  // chunk plan
  uint32_t nch;
  uint64_t need;
  uint64_t cw = 0;  // column chunk width (one stripe)
  uint32_t cs = 0;  // stripes per chunk
  if (S == 1) {
    // >= 2 KB per row and chunk: the 2D copies' DMA rate drops with shorter rows (config 5, one
    // box: 4 chunks of 2 KB 11.4 ms per step, 8 of 1 KB 12.0, 2 of 4 KB 13.4)
    const uint64_t max_chunks = std::max<uint64_t>(1, t / 2048);
    nch = static_cast<uint32_t>(std::min<uint64_t>(chunks, max_chunks));
    cw = (t / nch + 63) / 64 * 64;  // 64-B slices keep the SMEM variant eligible
    nch = static_cast<uint32_t>((t + cw - 1) / cw);
    need = rows * t;  // one full-size set: chunks write disjoint columns
  } else {
    nch = std::min(S, chunks);
    cs = (S + nch - 1) / nch;
    nch = (S + cs - 1) / cs;
    need = std::min<uint64_t>(nch, 2) * cs * rows * t;  // one set per stream in use
  }
  const uint64_t set_bytes = static_cast<uint64_t>(cs) * rows * t;  // S > 1: one staging set
  // a new call starts after everything the previous one issued (its chunking may differ)
  for (int j = 0; j < 2; ++j) {
    if ((e = cudaStreamWaitEvent(c.st[j], c.done[0], 0)) != cudaSuccess) return io_fail(e, "cudaStreamWaitEvent");
    if ((e = cudaStreamWaitEvent(c.st[j], c.done[1], 0)) != cudaSuccess) return io_fail(e, "cudaStreamWaitEvent");
  }
  if (need > c.bytes) {
    cudaStreamSynchronize(c.st[0]);
    cudaStreamSynchronize(c.st[1]);
    if (c.buf) cudaFree(c.buf);
    c.buf = nullptr;
    c.bytes = 0;
    if ((e = cudaMalloc(&c.buf, need)) != cudaSuccess) return io_fail(e, "cudaMalloc (host-encode staging)");
    c.bytes = need;
  }
  // the chunks start after the work already queued on the caller's stream
  if ((e = cudaEventRecord(c.start, stream)) != cudaSuccess) return io_fail(e, "cudaEventRecord");
  for (int j = 0; j < 2; ++j)
    if ((e = cudaStreamWaitEvent(c.st[j], c.start, 0)) != cudaSuccess) return io_fail(e, "cudaStreamWaitEvent");
  auto issue_chunk = [&](uint32_t i) -> fs_status {
    cudaStream_t st = c.st[i & 1];
    uint32_t L = 0;
    fs_status s;
    if (S == 1) {
      const uint64_t c0 = i * cw, c1 = std::min<uint64_t>(t, c0 + cw), w = c1 - c0;
      uint8_t *d = c.buf, *ck = c.buf + k * t, *y = c.buf + (k + p) * t;
      if ((e = cudaMemcpy2DAsync(d + c0, t, h_data + c0, t, w, k, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (data)");
      s = launch_encode(g, 1, d, k * t, p ? ck : nullptr, p * t, y, n * t, 0, g.prm.n, c0, c1, st, &L);
      if (s != FS_OK) return s;
      if (p && (e = cudaMemcpy2DAsync(h_checks + c0, t, ck + c0, t, w, p, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (checks)");
      if ((e = cudaMemcpy2DAsync(h_coded + c0, t, y + c0, t, w, n, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (coded)");
    } else {
      const uint32_t a = i * cs, b = std::min(S, a + cs), m = b - a;
      uint8_t *d = c.buf + (i & 1) * set_bytes, *ck = d + cs * k * t, *y = ck + cs * p * t;
      if ((e = cudaMemcpy2DAsync(d, k * t, h_data + a * data_stride, data_stride, k * t, m, cudaMemcpyHostToDevice,
                                 st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (data)");
      s = launch_encode(g, m, d, k * t, p ? ck : nullptr, p * t, y, n * t, 0, g.prm.n, 0, t, st, &L);
      if (s != FS_OK) return s;
      if (p && (e = cudaMemcpy2DAsync(h_checks + a * checks_stride, checks_stride, ck, p * t, p * t, m,
                                      cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (checks)");
      if ((e = cudaMemcpy2DAsync(h_coded + a * coded_stride, coded_stride, y, n * t, n * t, m, cudaMemcpyDeviceToHost,
                                 st)) != cudaSuccess)
        return io_fail(e, "cudaMemcpy2DAsync (coded)");
    }
    *launches += L;
    return FS_OK;
  };
  // every exit after this point first records done[] on both library streams and makes the
  // caller's stream wait for them, so chunks already queued when a later one fails are ordered
  // before anything the caller (or the next call) does with these buffers
  fs_status status = FS_OK;
  for (uint32_t i = 0; i < nch && status == FS_OK; ++i) status = issue_chunk(i);
  for (int j = 0; j < 2; ++j) {
    if ((e = cudaEventRecord(c.done[j], c.st[j])) != cudaSuccess) return io_fail(e, "cudaEventRecord");
    if ((e = cudaStreamWaitEvent(stream, c.done[j], 0)) != cudaSuccess) return io_fail(e, "cudaStreamWaitEvent");
  }
  return status;
}

}  // namespace fsb
