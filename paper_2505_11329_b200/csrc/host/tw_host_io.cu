// tw_host_io.cu -- K2 over HOST-resident activations as a three-stage
// pipeline: an H2D stream, a compute stream and a D2H stream, one chunk of
// rows per stage, R slots of device staging.  The H2D copy engine streams
// chunk k+1 while K2 runs on chunk k and the D2H engine drains chunk k-1
// (PCIe / C2C is full duplex, so both copy engines run at once).  This is the
// path the drop-in's host-matrix API and bench.py's `e2e` leg use.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
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
  // ~8 MiB chunks (8-16 MiB measured best on B200 over PCIe Gen5)
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

// ---- synchronous path for pageable host memory (the drop-in's std::vectors) --------
//
// cudaMemcpyAsync from pageable memory is staged by the driver one piece at a
// time on the calling thread (~5-10 GB/s, and it serialises the pipeline
// above).  Here a pool of host threads copies each chunk between the caller's
// memory and a pinned ring (scanning for NaN/Inf on the way in when asked),
// and the copy engines move only pinned memory:
//
//   iteration k:  [host] copy-out chunk k-R (after its D2H) ; copy-in chunk k
//                 [gpu ] H2D k | K2 k | D2H k   (three streams, as above)
//
// so the host copies of one chunk overlap the DMA and the kernel of the others.

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <vector>

namespace tw {
namespace {

inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#endif
}

// Fixed pool; run(n, f) calls f(0..n-1) across the workers and the caller.
// The staged copies call run() once per 8 MiB chunk, every ~0.2 ms, so idle
// workers spin for a while before sleeping on the condition variable, and the
// caller spins on the completion count before it sleeps: a futex wake-up per
// worker per chunk cost ~0.5 ms per call on these VMs (a 4 MiB staged copy
// took 0.78 ms, 32 MiB 2.7 ms).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // never destroyed (threads detached at exit)
    return *p;
  }
  int size() const { return static_cast<int>(threads_.size()) + 1; }
  void run(int n, const std::function<void(int)>& f) {
    job_ = &f;
    n_ = n;
    next_.store(0, std::memory_order_relaxed);
    done_.store(0, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);  // a worker between its check and its wait cannot miss this
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    const int want = static_cast<int>(threads_.size());
    for (int spins = 0; done_.load(std::memory_order_acquire) != want; ++spins) {
      if (spins < kCallerSpins) {
        cpu_relax();
      } else {
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait_for(lk, std::chrono::microseconds(100),
                          [&] { return done_.load(std::memory_order_acquire) == want; });
      }
    }
    job_ = nullptr;
  }

 private:
  static constexpr int kCallerSpins = 1 << 16;
  static constexpr std::chrono::microseconds kIdleSpin{500};
  HostPool() {
    // Half the hardware threads (the caller is one of them): the staging
    // copies are host-memory-bandwidth work that saturates well before every
    // core copies, and the spare cores keep the caller's other threads (the
    // drop-in's result fills, the CUDA driver's) off the pool's cores.  On the
    // 16-vCPU B200 VMs, interleaved A/B (profiles/dropin_fill_ab_r02.txt):
    // the drop-in rmsnorm_residual 40-43 ms with 16 threads, 30.6-31.4 with 8;
    // the TP = 2 fused op 8.7-9.0 vs 8.2-8.4 ms.  TW_HOST_THREADS overrides.
    unsigned hw = std::max(2u, std::thread::hardware_concurrency() / 2);
    if (const char* e = std::getenv("TW_HOST_THREADS")) {
      const int v = std::atoi(e);
      if (v >= 1) hw = static_cast<unsigned>(v);
    }
    const int workers = static_cast<int>(std::min(32u, hw)) - 1;
    for (int i = 0; i < std::max(0, workers); ++i)
      threads_.emplace_back([this] { loop(); });
    for (auto& t : threads_) t.detach();
  }
  void work() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*job_)(i);
  }
  void loop() {
    unsigned seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      int spins = 0;
      while (gen_.load(std::memory_order_acquire) == seen) {
        if ((++spins & 255) == 0 && std::chrono::steady_clock::now() - t0 > kIdleSpin) {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
          break;
        }
        cpu_relax();
      }
      seen = gen_.load(std::memory_order_acquire);
      work();
      if (done_.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<int>(threads_.size())) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0;
  std::atomic<unsigned> gen_{0};
  std::atomic<int> next_{0}, done_{0};
};

// Copy `bytes` and report whether any element is NaN/Inf (exponent all ones).
bool copy_check(void* dst, const void* src, size_t bytes, bool bf16, bool check) {
  std::memcpy(dst, src, bytes);
  if (!check) return false;
  if (bf16) {
    const uint16_t* v = static_cast<const uint16_t*>(dst);
    uint32_t bad = 0;
    for (size_t i = 0, n = bytes / 2; i < n; ++i) bad |= (v[i] & 0x7F80u) == 0x7F80u;
    return bad != 0;
  }
  const uint32_t* v = static_cast<const uint32_t*>(dst);
  uint32_t bad = 0;
  for (size_t i = 0, n = bytes / 4; i < n; ++i) bad |= (v[i] & 0x7F800000u) == 0x7F800000u;
  return bad != 0;
}

struct PinnedRing {
  int device = -1;
  size_t chunk = 0;
  void* h[kSlots][4] = {};  // pinned in, res, out, res_out
  cudaEvent_t drained[kSlots] = {};
};
PinnedRing g_ring[64];

tw_status ensure_ring(PinnedRing& g, int dev, size_t chunk) {
  if (g.device != dev) {
    g.device = dev;
    for (int i = 0; i < kSlots; ++i) {
      cudaError_t e = cudaEventCreateWithFlags(&g.drained[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "host_sync: events");
    }
  }
  if (g.chunk < chunk) {
    for (int i = 0; i < kSlots; ++i)
      for (int j = 0; j < 4; ++j) {
        if (g.h[i][j]) cudaFreeHost(g.h[i][j]);
        g.h[i][j] = nullptr;
        cudaError_t e = cudaHostAlloc(&g.h[i][j], chunk, cudaHostAllocDefault);
        if (e != cudaSuccess) {
          g.chunk = 0;
          return cuda_fail(e, "host_sync: cudaHostAlloc");
        }
      }
    g.chunk = chunk;
  }
  return TW_OK;
}

}  // namespace
}  // namespace tw

extern "C" {

tw_status tw_rmsnorm_residual_host_sync(const void* h_input, const void* h_residual, void* h_residual_out,
                                        void* h_output, const float* h_weight, int64_t T, int64_t H, float eps,
                                        tw_dtype dtype, unsigned flags) {
  return tw_rmsnorm_residual_host_sync_gated(h_input, h_residual, h_residual_out, h_output, h_weight, T, H, eps,
                                             dtype, flags, nullptr, 0);
}

tw_status tw_rmsnorm_residual_host_sync_gated(const void* h_input, const void* h_residual, void* h_residual_out,
                                              void* h_output, const float* h_weight, int64_t T, int64_t H,
                                              float eps, tw_dtype dtype, unsigned flags, const int64_t* rows_ready,
                                              int n_ready) {
  clear_error();
  if (n_ready < 0 || (n_ready > 0 && !rows_ready))
    return fail(TW_ERR_DIMENSION, "rmsnorm_residual_host_sync: bad rows_ready gate");
  if (T < 0 || H < 1) return fail(TW_ERR_DIMENSION, "rmsnorm_residual_host_sync: requires T >= 0 and H >= 1");
  if (!(eps > 0.0f) && eps != 0.0f)
    return fail(TW_ERR_NUMERIC, "rmsnorm_residual_host_sync: epsilon must be nonnegative");
  if (dtype != TW_BF16 && dtype != TW_F32) return fail(TW_ERR_CONFIG, "rmsnorm_residual_host_sync: unknown dtype");
  if (T == 0) return TW_OK;
  if (!h_input || !h_residual || !h_residual_out || !h_output || !h_weight)
    return fail(TW_ERR_DIMENSION, "rmsnorm_residual_host_sync: null buffer");
  const bool bf16 = dtype == TW_BF16;
  const bool check = flags & TW_HOST_CHECK_FINITE;
  const size_t row = static_cast<size_t>(H) * (bf16 ? 2 : 4);
  const int64_t chunk_rows = std::min<int64_t>(T, std::max<int64_t>(1, static_cast<int64_t>((8u << 20) / row)));
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(TW_ERR_CONFIG, "rmsnorm_residual_host_sync: device index");
  std::lock_guard<std::mutex> lock(g_mu);
  HostIoCtx& c = g_ctx[dev];
  PinnedRing& g = g_ring[dev];
  const size_t cb = static_cast<size_t>(chunk_rows) * row;
  tw_status st = ensure(c, dev, cb, static_cast<size_t>(H) * sizeof(float));
  if (st == TW_OK) st = ensure_ring(g, dev, cb);
  if (st != TW_OK) return st;
  cudaError_t e = cudaSuccess;
  for (cudaStream_t s : {c.h2d, c.comp, c.d2h}) cudaStreamWaitEvent(s, c.done, 0);
  e = cudaMemcpyAsync(c.weight, h_weight, H * sizeof(float), cudaMemcpyHostToDevice, c.h2d);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.h2d);  // h_weight may be pageable and short-lived
  if (e != cudaSuccess) return cuda_fail(e, "host_sync: weight H2D");
  // on any failure after work was enqueued: let the in-flight copies and
  // kernels finish before returning, so no DMA still targets the pinned ring
  // or the device slots when the next call reuses them
  auto drain = [&](tw_status why) {
    for (cudaStream_t q : {c.h2d, c.comp, c.d2h}) cudaStreamSynchronize(q);
    return why;
  };
  HostPool& pool = HostPool::get();
  const int parts = pool.size();
  const char* hin = static_cast<const char*>(h_input);
  const char* hres = static_cast<const char*>(h_residual);
  char* hro = static_cast<char*>(h_residual_out);
  char* hout = static_cast<char*>(h_output);
  const int64_t K = (T + chunk_rows - 1) / chunk_rows;
  auto span = [&](int64_t k, size_t* off, size_t* nb) {
    const int64_t r0 = k * chunk_rows, n = std::min(chunk_rows, T - r0);
    *off = static_cast<size_t>(r0) * row;
    *nb = static_cast<size_t>(n) * row;
  };
  // parallel copy of one chunk's two matrices, split in `parts` x 2 pieces
  auto pcopy = [&](char* d0, const char* s0, char* d1, const char* s1, size_t nb, bool chk) {
    std::atomic<bool> bad{false};
    const size_t elem = bf16 ? 2 : 4;
    const size_t piece = ((nb / elem + parts - 1) / parts) * elem;
    pool.run(2 * parts, [&](int i) {
      const int m = i / parts;
      const size_t a = static_cast<size_t>(i % parts) * piece;
      if (a >= nb) return;
      const size_t n = std::min(piece, nb - a);
      if (copy_check((m ? d1 : d0) + a, (m ? s1 : s0) + a, n, bf16, chk)) bad.store(true);
    });
    return bad.load();
  };
  auto copy_out = [&](int64_t k) -> tw_status {
    const int s = static_cast<int>(k % kSlots);
    cudaError_t ee = cudaEventSynchronize(g.drained[s]);
    if (ee != cudaSuccess) return drain(cuda_fail(ee, "host_sync: D2H"));
    size_t off, nb;
    span(k, &off, &nb);
    // the caller may still be preparing the destination rows (the drop-in
    // value-initialises its result vectors on helper threads): wait until
    // every gate covers this chunk
    const int64_t need = std::min(T, (k + 1) * chunk_rows);
    for (int i = 0; i < n_ready; ++i)
      for (int spins = 0; __atomic_load_n(rows_ready + i, __ATOMIC_ACQUIRE) < need; ++spins)
        if (spins < 4096) cpu_relax(); else std::this_thread::yield();
    pcopy(hout + off, static_cast<const char*>(g.h[s][2]), hro + off, static_cast<const char*>(g.h[s][3]), nb,
          false);
    return TW_OK;
  };
  bool nonfinite = false;
  for (int64_t k = 0; k < K && !nonfinite; ++k) {
    const int s = static_cast<int>(k % kSlots);
    if (k >= kSlots && (st = copy_out(k - kSlots)) != TW_OK) return drain(st);  // also frees slot s's pinned in/out
    size_t off, nb;
    span(k, &off, &nb);
    const int64_t n = static_cast<int64_t>(nb / row);
    if (pcopy(static_cast<char*>(g.h[s][0]), hin + off, static_cast<char*>(g.h[s][1]), hres + off, nb, check)) {
      nonfinite = true;
      break;
    }
    void** b = c.buf[s];
    if ((e = cudaMemcpyAsync(b[0], g.h[s][0], nb, cudaMemcpyHostToDevice, c.h2d)) != cudaSuccess ||
        (e = cudaMemcpyAsync(b[1], g.h[s][1], nb, cudaMemcpyHostToDevice, c.h2d)) != cudaSuccess)
      return drain(cuda_fail(e, "host_sync: H2D"));
    cudaEventRecord(c.loaded[s], c.h2d);
    cudaStreamWaitEvent(c.comp, c.loaded[s], 0);
    // (slot s's previous chunk, k - kSlots, was drained: copy_out synchronised on it)
    st = tw_rmsnorm_residual(b[0], b[1], b[3], b[2], static_cast<const float*>(c.weight), n, H, eps, dtype, 0, c.comp);
    if (st != TW_OK) return drain(st);
    cudaEventRecord(c.computed[s], c.comp);
    cudaStreamWaitEvent(c.d2h, c.computed[s], 0);
    if ((e = cudaMemcpyAsync(g.h[s][2], b[2], nb, cudaMemcpyDeviceToHost, c.d2h)) != cudaSuccess ||
        (e = cudaMemcpyAsync(g.h[s][3], b[3], nb, cudaMemcpyDeviceToHost, c.d2h)) != cudaSuccess)
      return drain(cuda_fail(e, "host_sync: D2H"));
    cudaEventRecord(g.drained[s], c.d2h);
  }
  if (nonfinite) return drain(fail(TW_ERR_NUMERIC, "TokenMatrix contains NaN/Inf"));
  for (int64_t k = std::max<int64_t>(0, K - kSlots); k < K; ++k)
    if ((st = copy_out(k)) != TW_OK) return drain(st);
  cudaEventRecord(c.done, c.d2h);  // every chunk drained (copy_out synchronised on each)
  return TW_OK;
}

}  // extern "C"

// ---- staged host <-> device copies (the drop-in's RankGroup matrices) ---------------

namespace tw {
namespace {

constexpr size_t kStageChunk = 8u << 20;

// The device owning a device pointer (-1: not device memory).
int device_of(const void* p) {
  cudaPointerAttributes a = {};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return a.type == cudaMemoryTypeDevice ? a.device : -1;
}

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

// Parallel copy of `nb` bytes split over the pool (optionally scanning for NaN/Inf).
bool pool_copy(HostPool& pool, char* dst, const char* src, size_t nb, size_t elem, bool bf16, bool check) {
  const int parts = pool.size();
  std::atomic<bool> bad{false};
  const size_t piece = ((nb / elem + parts - 1) / parts) * elem;
  pool.run(parts, [&](int i) {
    const size_t a = static_cast<size_t>(i) * piece;
    if (a >= nb) return;
    if (copy_check(dst + a, src + a, std::min(piece, nb - a), bf16, check)) bad.store(true);
  });
  return bad.load();
}

}  // namespace
}  // namespace tw

extern "C" {

tw_status tw_memcpy_h2d_staged(void* d_dst, const void* h_src, size_t bytes, tw_dtype dtype, unsigned flags,
                               int* nonfinite) {
  clear_error();
  if (nonfinite) *nonfinite = 0;
  if (bytes == 0) return TW_OK;
  if (!d_dst || !h_src) return fail(TW_ERR_DIMENSION, "memcpy_h2d_staged: null buffer");
  if (dtype != TW_BF16 && dtype != TW_F32) return fail(TW_ERR_CONFIG, "memcpy_h2d_staged: unknown dtype");
  const size_t elem = dtype == TW_BF16 ? 2 : 4;
  if (bytes % elem) return fail(TW_ERR_DIMENSION, "memcpy_h2d_staged: size not a multiple of the element");
  const int dev = device_of(d_dst);
  if (dev < 0 || dev >= 64) return fail(TW_ERR_CONFIG, "memcpy_h2d_staged: destination is not device memory");
  DeviceScope scope(dev);
  std::lock_guard<std::mutex> lock(g_mu);
  HostIoCtx& c = g_ctx[dev];
  PinnedRing& g = g_ring[dev];
  tw_status st = ensure(c, dev, 0, 0);
  if (st == TW_OK) st = ensure_ring(g, dev, kStageChunk);
  if (st != TW_OK) return st;
  // cudaMemcpy's ordering: after the legacy stream's prior work on this device
  cudaEventRecord(c.start, cudaStreamLegacy);
  cudaStreamWaitEvent(c.h2d, c.start, 0);
  HostPool& pool = HostPool::get();
  const bool check = flags & TW_HOST_CHECK_FINITE;
  bool bad = false;
  const char* src = static_cast<const char*>(h_src);
  char* dst = static_cast<char*>(d_dst);
  const size_t K = (bytes + kStageChunk - 1) / kStageChunk;
  for (size_t k = 0; k < K; ++k) {
    const int s = static_cast<int>(k % kSlots);
    const size_t off = k * kStageChunk, nb = std::min(kStageChunk, bytes - off);
    if (k >= static_cast<size_t>(kSlots)) {
      cudaError_t e = cudaEventSynchronize(g.drained[s]);  // the slot's previous DMA has read it
      if (e != cudaSuccess) return cuda_fail(e, "memcpy_h2d_staged: H2D");
    }
    bad |= pool_copy(pool, static_cast<char*>(g.h[s][0]), src + off, nb, elem, dtype == TW_BF16, check);
    cudaError_t e = cudaMemcpyAsync(dst + off, g.h[s][0], nb, cudaMemcpyHostToDevice, c.h2d);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(c.h2d);
      return cuda_fail(e, "memcpy_h2d_staged: H2D");
    }
    cudaEventRecord(g.drained[s], c.h2d);
  }
  cudaError_t e = cudaStreamSynchronize(c.h2d);
  if (e != cudaSuccess) return cuda_fail(e, "memcpy_h2d_staged: H2D");
  if (nonfinite) *nonfinite = bad ? 1 : 0;
  return TW_OK;
}

tw_status tw_memcpy_d2h_staged(void* h_dst, const void* d_src, size_t bytes) {
  clear_error();
  if (bytes == 0) return TW_OK;
  if (!h_dst || !d_src) return fail(TW_ERR_DIMENSION, "memcpy_d2h_staged: null buffer");
  const int dev = device_of(d_src);
  if (dev < 0 || dev >= 64) return fail(TW_ERR_CONFIG, "memcpy_d2h_staged: source is not device memory");
  DeviceScope scope(dev);
  std::lock_guard<std::mutex> lock(g_mu);
  HostIoCtx& c = g_ctx[dev];
  PinnedRing& g = g_ring[dev];
  tw_status st = ensure(c, dev, 0, 0);
  if (st == TW_OK) st = ensure_ring(g, dev, kStageChunk);
  if (st != TW_OK) return st;
  cudaEventRecord(c.start, cudaStreamLegacy);
  cudaStreamWaitEvent(c.d2h, c.start, 0);
  HostPool& pool = HostPool::get();
  const char* src = static_cast<const char*>(d_src);
  char* dst = static_cast<char*>(h_dst);
  const size_t K = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t k) -> cudaError_t {
    const int s = static_cast<int>(k % kSlots);
    const size_t off = k * kStageChunk, nb = std::min(kStageChunk, bytes - off);
    cudaError_t e = cudaMemcpyAsync(g.h[s][2], src + off, nb, cudaMemcpyDeviceToHost, c.d2h);
    if (e == cudaSuccess) e = cudaEventRecord(g.drained[s], c.d2h);
    return e;
  };
  for (size_t k = 0; k < std::min(K, static_cast<size_t>(kSlots)); ++k) {
    cudaError_t e = issue(k);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(c.d2h);
      return cuda_fail(e, "memcpy_d2h_staged: D2H");
    }
  }
  for (size_t k = 0; k < K; ++k) {
    const int s = static_cast<int>(k % kSlots);
    const size_t off = k * kStageChunk, nb = std::min(kStageChunk, bytes - off);
    cudaError_t e = cudaEventSynchronize(g.drained[s]);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(c.d2h);
      return cuda_fail(e, "memcpy_d2h_staged: D2H");
    }
    pool_copy(pool, dst + off, static_cast<const char*>(g.h[s][2]), nb, 1, false, false);
    if (k + kSlots < K && (e = issue(k + kSlots)) != cudaSuccess) {  // the slot is free again
      cudaStreamSynchronize(c.d2h);
      return cuda_fail(e, "memcpy_d2h_staged: D2H");
    }
  }
  return TW_OK;
}

}  // extern "C"
