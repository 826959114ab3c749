// tw_host_io.cu -- K2 over HOST-resident activations as a three-stage
// pipeline: an H2D stream, a compute stream and a D2H stream, one chunk of
// rows per stage, R slots of device staging.  The H2D copy engine streams
// chunk k+1 while K2 runs on chunk k and the D2H engine drains chunk k-1
// (PCIe / C2C is full duplex, so both copy engines run at once).  This is the
// path the drop-in's host-matrix API and bench.py's `e2e` leg use.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "tw_internal.h"

namespace tw {
namespace {

constexpr int kSlots = 4;

struct HostIoCtx {
  int device = -1;
  size_t chunk_bytes = 0;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t loaded[kSlots] = {}, computed[kSlots] = {}, drained[kSlots] = {};
  cudaEvent_t start = nullptr, finish_c = nullptr, finish_d = nullptr;
  // recorded on d2h after every call's last copy (d2h having joined comp):
  // the next call's three streams wait on it, so a call issued on another
  // caller stream cannot overwrite the weight or a staging slot the previous
  // call is still reading (the mutex only serialises enqueueing)
  cudaEvent_t done = nullptr;
  void* buf[kSlots][4] = {};  // in, res, out, res_out per slot
  void* weight = nullptr;
  size_t weight_bytes = 0;
};

std::mutex g_mu;
HostIoCtx g_ctx[64];

tw_status ensure(HostIoCtx& c, int dev, size_t chunk_bytes, size_t wbytes) {
  if (c.device != dev) {
    c.device = dev;
    cudaError_t e = cudaSuccess;
    for (cudaStream_t* s : {&c.h2d, &c.comp, &c.d2h})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&c.loaded[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.computed[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.drained[i], cudaEventDisableTiming);
    }
    for (cudaEvent_t* ev : {&c.start, &c.finish_c, &c.finish_d, &c.done})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host_io: streams/events");
  }
  if (c.chunk_bytes < chunk_bytes) {
    cudaDeviceSynchronize();
    for (int i = 0; i < kSlots; ++i)
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
  // ~8 MiB chunks (8-16 MiB measured best on B200 over PCIe Gen5, tools/e2e_probe.py)
  if (chunk_rows <= 0) chunk_rows = std::max<int64_t>(1, static_cast<int64_t>((8u << 20) / row));
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
  for (cudaStream_t s : {c.h2d, c.comp, c.d2h}) {
    cudaStreamWaitEvent(s, c.start, 0);
    cudaStreamWaitEvent(s, c.done, 0);  // the previous call on this device (no-op before the first)
  }
  e = cudaMemcpyAsync(c.weight, h_weight, H * sizeof(float), cudaMemcpyHostToDevice, c.h2d);
  if (e != cudaSuccess) return cuda_fail(e, "host_io: weight H2D");
  const char* hin = static_cast<const char*>(h_input);
  const char* hres = static_cast<const char*>(h_residual);
  char* hro = static_cast<char*>(h_residual_out);
  char* hout = static_cast<char*>(h_output);
  int64_t k = 0;
  for (int64_t r0 = 0; r0 < T; r0 += chunk_rows, ++k) {
    const int slot = static_cast<int>(k % kSlots);
    const int64_t n = std::min(chunk_rows, T - r0);
    const size_t off = static_cast<size_t>(r0) * row, nb = static_cast<size_t>(n) * row;
    void** b = c.buf[slot];
    // stage 1: H2D, once the slot's previous chunk has drained
    if (k >= kSlots) cudaStreamWaitEvent(c.h2d, c.drained[slot], 0);
    if ((e = cudaMemcpyAsync(b[0], hin + off, nb, cudaMemcpyHostToDevice, c.h2d)) != cudaSuccess ||
        (e = cudaMemcpyAsync(b[1], hres + off, nb, cudaMemcpyHostToDevice, c.h2d)) != cudaSuccess)
      return cuda_fail(e, "host_io: H2D");
    cudaEventRecord(c.loaded[slot], c.h2d);
    // stage 2: the kernel
    cudaStreamWaitEvent(c.comp, c.loaded[slot], 0);
    st = tw_rmsnorm_residual(b[0], b[1], b[3], b[2], static_cast<const float*>(c.weight), n, H, eps, dtype, 0, c.comp);
    if (st != TW_OK) return st;
    cudaEventRecord(c.computed[slot], c.comp);
    // stage 3: D2H
    cudaStreamWaitEvent(c.d2h, c.computed[slot], 0);
    if ((e = cudaMemcpyAsync(hout + off, b[2], nb, cudaMemcpyDeviceToHost, c.d2h)) != cudaSuccess ||
        (e = cudaMemcpyAsync(hro + off, b[3], nb, cudaMemcpyDeviceToHost, c.d2h)) != cudaSuccess)
      return cuda_fail(e, "host_io: D2H");
    cudaEventRecord(c.drained[slot], c.d2h);
  }
  cudaEventRecord(c.finish_c, c.comp);
  cudaEventRecord(c.finish_d, c.d2h);
  cudaStreamWaitEvent(c.d2h, c.finish_c, 0);
  cudaEventRecord(c.done, c.d2h);
  cudaStreamWaitEvent(caller, c.finish_c, 0);
  cudaStreamWaitEvent(caller, c.finish_d, 0);
  return TW_OK;
}

}  // extern "C"
