// tw_flat.cuh -- K2 "flat" engine: one CTA of up to 1024 threads owns one row
// at a time (VPT 16-byte vectors per thread), two CTAs per SM, 32 registers,
// one __syncthreads per row (double-buffered partial sums).  No warp
// specialisation, no shared-memory staging: the row's loads are register
// loads issued all at once, like a plain streaming copy -- the shape that
// reaches the per-SM copy rate (~95 GB/s/SM measured, tools/probe/smbw.cu)
// when only part of the GPU is available or the batch is short.
#pragma once

#include <cstdint>
#include <type_traits>

#include "tw_rownorm.cuh"

namespace tw {

struct FlatParams {
  const void* in;
  const void* res_in;
  void* res_out;
  void* out;
  const float* weight;
  long long T, H;
  int V;  // 16-byte vectors per row
  float eps;
};

template <class E, int VPT>
__global__ void __launch_bounds__(1024, 2) k2_flat_kernel(const __grid_constant__ FlatParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Raw = typename VT::Raw;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  __shared__ Acc part[2][32];
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int nwarps = nthreads >> 5;
  int parity = 0;
  for (long long t = blockIdx.x; t < p.T; t += gridDim.x, parity ^= 1) {
    const long long rowe = t * p.H;
    Raw xr[VPT], rr[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = tid + k * nthreads;
      if (c < p.V) {
        xr[k] = VT::load_stream(p.in, rowe + static_cast<long long>(c) * N);
        rr[k] = VT::load_stream(p.res_in, rowe + static_cast<long long>(c) * N);
      }
    }
    Acc ss = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = tid + k * nthreads;
      if (c < p.V) {
        float x[N], r[N];
        VT::unpack(xr[k], x);
        VT::unpack(rr[k], r);
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = x[j] + r[j];
        rr[k] = VT::pack(r);
        VT::unpack(rr[k], r);
#pragma unroll
        for (int j = 0; j < N; ++j) ss += static_cast<Acc>(r[j]) * static_cast<Acc>(r[j]);
        VT::store(p.res_out, rowe + static_cast<long long>(c) * N, rr[k]);
      }
    }
    ss = warp_sum(ss);
    if ((tid & 31) == 0) part[parity][tid >> 5] = ss;
    __syncthreads();
    Acc total = 0;
    for (int w = 0; w < nwarps; ++w) total += part[parity][w];
    const float inv = 1.0f / sqrtf(static_cast<float>(total / static_cast<Acc>(p.H)) + p.eps);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = tid + k * nthreads;
      if (c < p.V) {
        float w[N], o[N];
        load_weight<N>(p.weight, static_cast<long long>(c) * N, w);
        VT::unpack(rr[k], o);
#pragma unroll
        for (int j = 0; j < N; ++j) o[j] = o[j] * inv * w[j];
        VT::store(p.out, rowe + static_cast<long long>(c) * N, VT::pack(o));
      }
    }
  }
}

}  // namespace tw
