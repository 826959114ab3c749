// k2floor.cu -- what does an event pair around ONE launch measure at K2's
// short-batch sizes (T = 256..4096, H = 8192 bf16) after an L2 flush?
// Variants (median of 50, write+read 256 MiB flush before each):
//   empty1     <<<1, 32>>> empty kernel (event + launch overhead)
//   emptyfull  <<<148, 544, 197 KB smem>>> empty kernel (K2's launch shape)
//   addU       streaming r' = x + r, out = r' (K2's traffic, no row reduction),
//              register path, 2 x 1024-thread CTAs per SM, U 16-B vectors in flight per thread per operand
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o k2floor k2floor.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void empty_kernel() {}

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

__device__ __forceinline__ uint4 add8(uint4 a, uint4 b) {
  uint4 o;
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&b);
  __nv_bfloat162* z = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
  for (int i = 0; i < 4; ++i) z[i] = __hadd2(x[i], y[i]);
  return o;
}

template <int U>
__global__ void __launch_bounds__(1024) add_stream(const uint4* __restrict__ x, const uint4* __restrict__ r,
                                                   uint4* __restrict__ ro, uint4* __restrict__ o, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i < n; i += U * stride) {
    uint4 a[U], b[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i + k * stride < n) {
        a[k] = __ldcs(x + i + k * stride);
        b[k] = __ldcs(r + i + k * stride);
      }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i + k * stride < n) {
        uint4 s = add8(a[k], b[k]);
        __stcs(ro + i + k * stride, s);
        __stcs(o + i + k * stride, s);
      }
  }
}

int main() {
  const size_t H = 8192;
  const size_t Tmax = 16384;
  const size_t bytes = Tmax * H * 2;
  uint4 *x, *r, *ro, *o, *fl;
  uint32_t* sink;
  const size_t flbytes = 256ull << 20;
  cudaMalloc(&x, bytes);
  cudaMalloc(&r, bytes);
  cudaMalloc(&ro, bytes);
  cudaMalloc(&o, bytes);
  cudaMalloc(&fl, flbytes);
  cudaMalloc(&sink, 4);
  cudaMemset(x, 0, bytes);
  cudaMemset(r, 0, bytes);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 197 * 1024);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  auto flush = [&](int it) {
    fill_kernel<<<nsm * 4, 1024>>>(fl, flbytes / 16, it);
    read_kernel<<<nsm * 4, 1024>>>(fl, flbytes / 16, sink);
  };
  auto timeit = [&](auto fn) {
    std::vector<float> ts;
    for (int it = 0; it < 55; ++it) {
      flush(it);
      cudaEventRecord(s);
      fn();
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms = 0;
      cudaEventElapsedTime(&ms, s, e);
      if (it >= 5) ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
  };
  printf("empty1 %.2f us\n", timeit([&] { empty_kernel<<<1, 32>>>(); }));
  printf("emptyfull %.2f us\n", timeit([&] { empty_kernel<<<nsm, 544, 197 * 1024>>>(); }));
  for (size_t T : {256, 1024, 2048, 4096, 8192, 16384}) {
    const size_t n = T * H * 2 / 16;
    const double alg = 4.0 * T * H * 2;
    float t1 = timeit([&] { add_stream<1><<<nsm * 2, 1024>>>(x, r, ro, o, n); });
    float t2 = timeit([&] { add_stream<2><<<nsm * 2, 1024>>>(x, r, ro, o, n); });
    float t4 = timeit([&] { add_stream<4><<<nsm * 2, 1024>>>(x, r, ro, o, n); });
    printf("T=%zu add U1 %.2f us (%.0f GB/s)  U2 %.2f (%.0f)  U4 %.2f (%.0f)\n", T, t1, alg / t1 / 1e3, t2,
           alg / t2 / 1e3, t4, alg / t4 / 1e3);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
