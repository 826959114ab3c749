// pcie_zc.cu -- zero-copy PCIe probe: SM loads/stores straight to pinned host
// memory (UVA) vs the copy engines, one direction and both at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_zc pcie_zc.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e_));                           \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

// dst[i] = src[i] over n uint4, grid-stride, `unroll` independent loads in flight.
template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  const size_t N = 256ull << 20;
  void *h_in, *h_out, *d_a, *d_b;
  CK(cudaHostAlloc(&h_in, N, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_out, N, cudaHostAllocMapped));
  CK(cudaMalloc(&d_a, N));
  CK(cudaMalloc(&d_b, N));
  memset(h_in, 1, N);
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long n = N / 16;
  auto timeit = [&](auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3 / 1e3;
  };
  int grids[] = {64, 148, 296, 592};
  for (int g : grids) {
    double t = timeit([&] { copy_kernel<4><<<g, 512>>>((const uint4*)h_in, (uint4*)d_a, n); });
    printf("zc read  host->dev grid %4d: %.1f GB/s\n", g, N / t / 1e9);
    t = timeit([&] { copy_kernel<4><<<g, 512>>>((const uint4*)d_a, (uint4*)h_out, n); });
    printf("zc write dev->host grid %4d: %.1f GB/s\n", g, N / t / 1e9);
    t = timeit([&] { copy_kernel<4><<<g, 512>>>((const uint4*)h_in, (uint4*)h_out, n); });
    printf("zc host->host (both dirs) grid %4d: %.1f GB/s each\n", g, N / t / 1e9);
    t = timeit([&] {
      copy_kernel<4><<<g / 2 > 0 ? g / 2 : 1, 512, 0, s1>>>((const uint4*)h_in, (uint4*)d_a, n);
      copy_kernel<4><<<g / 2 > 0 ? g / 2 : 1, 512, 0, s2>>>((const uint4*)d_b, (uint4*)h_out, n);
      cudaStreamSynchronize(s1);
      cudaStreamSynchronize(s2);
    });
    printf("zc read || write (2 streams) grid %4d: %.1f GB/s each\n", g, N / t / 1e9);
  }
  double t = timeit([&] {
    cudaMemcpyAsync(d_a, h_in, N, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_out, d_b, N, cudaMemcpyDeviceToHost, s2);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
  });
  printf("copy engines H2D || D2H: %.1f GB/s each\n", N / t / 1e9);
  t = timeit([&] { cudaMemcpyAsync(d_a, h_in, N, cudaMemcpyHostToDevice, s1); cudaStreamSynchronize(s1); });
  printf("copy engine H2D: %.1f GB/s\n", N / t / 1e9);
  t = timeit([&] { cudaMemcpyAsync(h_out, d_b, N, cudaMemcpyDeviceToHost, s1); cudaStreamSynchronize(s1); });
  printf("copy engine D2H: %.1f GB/s\n", N / t / 1e9);
  // mixed: copy engine H2D || zero-copy writes D2H
  t = timeit([&] {
    cudaMemcpyAsync(d_a, h_in, N, cudaMemcpyHostToDevice, s1);
    copy_kernel<4><<<148, 512, 0, s2>>>((const uint4*)d_b, (uint4*)h_out, n);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
  });
  printf("CE H2D || zc D2H: %.1f GB/s each\n", N / t / 1e9);
  t = timeit([&] {
    copy_kernel<4><<<148, 512, 0, s1>>>((const uint4*)h_in, (uint4*)d_a, n);
    cudaMemcpyAsync(h_out, d_b, N, cudaMemcpyDeviceToHost, s2);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
  });
  printf("zc H2D || CE D2H: %.1f GB/s each\n", N / t / 1e9);
  return 0;
}
