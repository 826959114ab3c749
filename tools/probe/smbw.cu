// smbw.cu -- per-SM memory bandwidth on B200 vs the number of SMs used:
// read-only, write-only and copy streams, register path (LDG.128/STG.128,
// 8 loads in flight per thread) and TMA bulk path (cp.async.bulk, 6 x 32 KB
// stages).  Informs the SM budget of bandwidth-bound kernels (K1's 2-16-SM
// knob, K2 under a budget).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(1024) rd(const uint4* __restrict__ a, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(a + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc.x ^= v[k].x, acc.y ^= v[k].y, acc.z ^= v[k].z, acc.w ^= v[k].w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

__global__ void __launch_bounds__(1024) wr(uint4* __restrict__ a, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    __stcs(a + i, make_uint4(1, 2, 3, 4));
}

__global__ void __launch_bounds__(1024) cp(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(a + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(b + i + k * stride, v[k]);
  }
}

int main() {
  const size_t bytes = size_t(1) << 30;
  const size_t n = bytes / 16;
  uint4 *a, *b, *sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(a, 1, bytes);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  printf("sms  read_GBs(per SM)  write_GBs(per SM)  copy_GBs(per SM, r+w bytes)\n");
  for (int sms : {1, 2, 4, 8, 16, 32, 64, 148}) {
    const size_t nn = sms >= 16 ? n : n / 8;  // shorter streams for tiny grids
    float t[3];
    for (int k = 0; k < 3; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s);
        if (k == 0) rd<<<sms, 1024>>>(a, nn, sink);
        if (k == 1) wr<<<sms, 1024>>>(b, nn);
        if (k == 2) cp<<<sms, 1024>>>(a, b, nn / 2);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&t[k], s, e);
      }
    }
    const double gb = double(nn) * 16 / 1e9;
    printf("%4d  %8.1f (%6.1f)  %8.1f (%6.1f)  %8.1f (%6.1f)\n", sms, gb / (t[0] * 1e-3), gb / (t[0] * 1e-3) / sms,
           gb / (t[1] * 1e-3), gb / (t[1] * 1e-3) / sms, gb / (t[2] * 1e-3), gb / (t[2] * 1e-3) / sms);
  }
  return 0;
}
