// tw_host_io.cu -- K2 over HOST-resident activations: the row range is cut
// into chunks and pipelined over a ring of streams so that the H2D copy of
// chunk k+1, the kernel on chunk k and the D2H copy of chunk k-1 overlap
// (PCIe / C2C is full duplex: both copy engines run at once).  This is the
// path the drop-in's host-matrix API and bench.py's `e2e` leg use.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "tw_internal.h"

namespace tw {
namespace {

constexpr int kRing = 3;

struct HostIoCtx {
  int device = -1;
  size_t chunk_bytes = 0;
  cudaStream_t s[kRing] = {};
  cudaEvent_t done[kRing] = {};
  cudaEvent_t start = nullptr;
  void* buf[kRing][4] = {};  // in, res, out, res_out per slot
  void* weight = nullptr;
  size_t weight_bytes = 0;
};

std::mutex g_mu;
HostIoCtx g_ctx[64];

tw_status ensure(HostIoCtx& c, int dev, size_t chunk_bytes, size_t wbytes) {
  if (c.device != dev) {
    c.device = dev;
    for (int i = 0; i < kRing; ++i) {
      cudaError_t e = cudaStreamCreateWithFlags(&c.s[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.done[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "host_io: stream/event");
    }
    cudaError_t e = cudaEventCreateWithFlags(&c.start, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host_io: event");
  }
  if (c.chunk_bytes < chunk_bytes) {
    cudaDeviceSynchronize();
    for (int i = 0; i < kRing; ++i)
      for (int j = 0; j < 4; ++j) {
        if (c.buf[i][j]) cudaFree(c.buf[i][j]);
        c.buf[i][j] = nullptr;
        cudaError_t e = cudaMalloc(&c.buf[i][j], chunk_bytes);
        if (e != cudaSuccess) {
          c.chunk_bytes = 0;
          return cuda_fail(e, "host_io: cudaMalloc");
        }
      }
    c.chunk_bytes = chunk_bytes;
  }
  if (c.weight_bytes < wbytes) {
    if (c.weight) cudaFree(c.weight);
    cudaError_t e = cudaMalloc(&c.weight, wbytes);
    if (e != cudaSuccess) {
      c.weight_bytes = 0;
      return cuda_fail(e, "host_io: cudaMalloc(weight)");
    }
    c.weight_bytes = wbytes;
  }
  return TW_OK;
}

}  // namespace
}  // namespace tw

using namespace tw;

extern "C" {

tw_status tw_rmsnorm_residual_host(const void* h_input, const void* h_residual, void* h_residual_out,
                                   void* h_output, const float* h_weight, int64_t T, int64_t H, float eps,
                                   tw_dtype dtype, int64_t chunk_rows, void* stream) {
  clear_error();
  if (T < 0 || H < 1) return fail(TW_ERR_DIMENSION, "rmsnorm_residual_host: requires T >= 0 and H >= 1");
  if (!(eps > 0.0f) && eps != 0.0f) return fail(TW_ERR_NUMERIC, "rmsnorm_residual_host: epsilon must be nonnegative");
  if (dtype != TW_BF16 && dtype != TW_F32) return fail(TW_ERR_CONFIG, "rmsnorm_residual_host: unknown dtype");
  if (T == 0) return TW_OK;
  if (!h_input || !h_residual || !h_residual_out || !h_output || !h_weight)
    return fail(TW_ERR_DIMENSION, "rmsnorm_residual_host: null buffer");
  const size_t row = static_cast<size_t>(H) * (dtype == TW_BF16 ? 2 : 4);
  if (chunk_rows <= 0) chunk_rows = std::max<int64_t>(1, static_cast<int64_t>((8u << 20) / row));  // ~8 MiB chunks
  chunk_rows = std::min<int64_t>(chunk_rows, T);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(TW_ERR_CONFIG, "rmsnorm_residual_host: device index");
  std::lock_guard<std::mutex> lock(g_mu);
  HostIoCtx& c = g_ctx[dev];
  tw_status st = ensure(c, dev, static_cast<size_t>(chunk_rows) * row, static_cast<size_t>(H) * sizeof(float));
  if (st != TW_OK) return st;
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaEventRecord(c.start, caller);
  if (e != cudaSuccess) return cuda_fail(e, "host_io: record");
  for (int i = 0; i < kRing; ++i) cudaStreamWaitEvent(c.s[i], c.start, 0);
  e = cudaMemcpyAsync(c.weight, h_weight, H * sizeof(float), cudaMemcpyHostToDevice, c.s[0]);
  if (e != cudaSuccess) return cuda_fail(e, "host_io: weight H2D");
  cudaEvent_t wready = c.done[0];
  cudaEventRecord(wready, c.s[0]);
  for (int i = 1; i < kRing; ++i) cudaStreamWaitEvent(c.s[i], wready, 0);
  const char* hin = static_cast<const char*>(h_input);
  const char* hres = static_cast<const char*>(h_residual);
  char* hro = static_cast<char*>(h_residual_out);
  char* hout = static_cast<char*>(h_output);
  int64_t k = 0;
  for (int64_t r0 = 0; r0 < T; r0 += chunk_rows, ++k) {
    const int slot = static_cast<int>(k % kRing);
    const int64_t n = std::min(chunk_rows, T - r0);
    const size_t off = static_cast<size_t>(r0) * row, nb = static_cast<size_t>(n) * row;
    cudaStream_t s = c.s[slot];
    void** b = c.buf[slot];
    if ((e = cudaMemcpyAsync(b[0], hin + off, nb, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(b[1], hres + off, nb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "host_io: H2D");
    st = tw_rmsnorm_residual(b[0], b[1], b[3], b[2], static_cast<const float*>(c.weight), n, H, eps, dtype, 0, s);
    if (st != TW_OK) return st;
    if ((e = cudaMemcpyAsync(hout + off, b[2], nb, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(hro + off, b[3], nb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "host_io: D2H");
  }
  for (int i = 0; i < kRing; ++i) {
    cudaEventRecord(c.done[i], c.s[i]);
    cudaStreamWaitEvent(caller, c.done[i], 0);
  }
  return TW_OK;
}

}  // extern "C"
