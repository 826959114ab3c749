// k2trace.cu -- per-CTA timeline of K2's TMA engine (k2_tma_kernel, the
// product kernel built with TW_K2_TRACE) at a short batch, after an L2 flush:
// launch skew, weights-in-registers, each row's load issue / arrival / store
// issue, and the CTA's end, from %globaltimer (ns).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTW_K2_TRACE \
//      -I../../paper_2505_11329_b200/csrc -o k2trace k2trace.cu
//   ./k2trace T [lookahead] [groups] [threads per row group]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels/tw_bulk.cuh"

__global__ void fill_kernel(uint4* p, size_t n, uint32_t v) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
__global__ void read_kernel(const uint4* p, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    acc ^= p[i].x;
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const long long T = argc > 1 ? atoll(argv[1]) : 1024;
  const int la = argc > 2 ? atoi(argv[2]) : 0;
  const int G = argc > 3 ? atoi(argv[3]) : 2;
  const int TPR = argc > 4 ? atoi(argv[4]) : 256;
  const long long H = 8192;
  const size_t bytes = size_t(T) * H * 2;
  void *x, *r, *ro, *o;
  float* w;
  uint4* fl;
  uint32_t* sink;
  const size_t flbytes = 256ull << 20;
  cudaMalloc(&x, bytes);
  cudaMalloc(&r, bytes);
  cudaMalloc(&ro, bytes);
  cudaMalloc(&o, bytes);
  cudaMalloc(&w, H * 4);
  cudaMalloc(&fl, flbytes);
  cudaMalloc(&sink, 4);
  cudaMemset(x, 0, bytes);
  cudaMemset(r, 0, bytes);
  cudaMemset(w, 0, H * 4);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  tw::BulkParams p = {};
  p.in = x;
  p.res_in = r;
  p.res_out = ro;
  p.out = o;
  p.weight = w;
  p.T = T;
  p.H = H;
  p.V = int(H / 8);
  p.tpr = TPR;
  p.groups = G;
  p.row_bytes = uint32_t(H * 2);
  p.stages = int(std::min<size_t>(8, (200 * 1024) / (2ull * p.row_bytes)));
  p.lookahead = la;
  p.eps = 1e-5f;
  auto fn = G == 2 ? (TPR == 512 ? tw::k2_tma_kernel<uint16_t, 2, 2> : tw::k2_tma_kernel<uint16_t, 4, 2>)
                   : (TPR == 512 ? tw::k2_tma_kernel<uint16_t, 2, 1> : tw::k2_tma_kernel<uint16_t, 4, 1>);
  const size_t smem = size_t(p.stages) * 2 * p.row_bytes + 2 * p.stages * 8 + 2 * G * (TPR / 32) * 8;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int grid = int(std::min<long long>(T, nsm));
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  std::vector<unsigned long long> tr(size_t(grid) * 64);
  std::vector<float> ts;
  unsigned long long* dtr = nullptr;
  cudaGetSymbolAddress(reinterpret_cast<void**>(&dtr), tw::k2_trace);
  for (int it = 0; it < 21; ++it) {
    cudaMemset(dtr, 0, tr.size() * 8);
    fill_kernel<<<nsm * 4, 1024>>>(fl, flbytes / 16, it);
    read_kernel<<<nsm * 4, 1024>>>(fl, flbytes / 16, sink);
    cudaEventRecord(s);
    fn<<<grid, G * TPR + 32, smem>>>(p);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms = 0;
    cudaEventElapsedTime(&ms, s, e);
    ts.push_back(ms * 1e3f);
  }
  cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
  printf("T=%lld la=%d G=%d stages=%d grid=%d status=%s event_us(last)=%.2f median=%.2f\n", T, la, G, p.stages, grid,
         cudaGetErrorString(cudaGetLastError()), ts.back(), [&] {
           auto v = ts;
           std::sort(v.begin(), v.end());
           return v[v.size() / 2];
         }());
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < grid; ++b) t0 = std::min(t0, tr[b * 64 + 0]);
  auto rel = [&](int b, int k) { return tr[b * 64 + k] ? (double)(tr[b * 64 + k] - t0) / 1e3 : -1.0; };
  // distribution summaries over CTAs
  auto stat = [&](const char* name, int k) {
    std::vector<double> v;
    for (int b = 0; b < grid; ++b)
      if (tr[b * 64 + k]) v.push_back(rel(b, k));
    if (v.empty()) return;
    std::sort(v.begin(), v.end());
    printf("  %-14s n=%3zu min %6.2f  med %6.2f  max %6.2f us\n", name, v.size(), v.front(), v[v.size() / 2],
           v.back());
  };
  stat("start", 0);
  stat("weights g0", 40);
  for (int i = 0; i < 8; ++i) {
    char nm[32];
    snprintf(nm, sizeof nm, "issue row %d", i);
    stat(nm, 1 + i);
  }
  for (int i = 0; i < 8; ++i) {
    char nm[32];
    snprintf(nm, sizeof nm, "arrive row %d", i);
    stat(nm, 10 + i);
  }
  for (int i = 0; i < 8; ++i) {
    char nm[32];
    snprintf(nm, sizeof nm, "store row %d", i);
    stat(nm, 20 + i);
  }
  for (int i = 0; i < 4; ++i) {
    const char* ph[4] = {"pass1 done", "inv ready", "pass2 done", "fenced+bar"};
    for (int k = 0; k < 4; ++k) {
      char nm[32];
      snprintf(nm, sizeof nm, "r%d %s", i, ph[k]);
      stat(nm, 44 + 4 * i + k);
    }
  }
  stat("end g0", 30);
  stat("end g1", 31);
  {
    std::vector<double> ends;
    for (int b = 0; b < grid; ++b) {
      double e = std::max(rel(b, 30), rel(b, 31));
      if (e > 0) ends.push_back(e);
    }
    std::sort(ends.begin(), ends.end());
    printf("  CTA end deciles:");
    for (int q = 0; q <= 10; ++q) printf(" %.1f", ends[std::min(ends.size() - 1, ends.size() * q / 10)]);
    printf("\n");
  }
  printf("  CTA 0 :");
  for (int k : {0, 40, 1, 2, 3, 4, 5, 6, 7, 10, 11, 12, 13, 14, 15, 16, 20, 21, 22, 23, 24, 25, 26, 30, 31})
    printf(" %d:%.2f", k, rel(0, k));
  printf("\n");
  return 0;
}
