// smcopy.cu -- how fast can ONE SM stream a copy-shaped workload (read 2 rows,
// write 2 rows per token, K2's traffic) when only a few SMs run?  The SM-
// budgeted boundary op (the weave on one GPU, K1's local traffic) is bound by
// this per-SM rate, not by HBM.  Variants:
//   lsu  U  C : register path, 1024-thread CTAs, U 16-B loads in flight per
//               thread, C CTAs per SM
//   tma  S  C : bulk engine only: G2S cp.async.bulk of 32 KB into an S-stage
//               ring, S2G cp.async.bulk of the same stage, C CTAs per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o smcopy smcopy.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int U>
__global__ void __launch_bounds__(1024) lsu_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldcs(a + i + k * stride);
#pragma unroll
    for (int k = 0; k < U; ++k) __stcs(b + i + k * stride, v[k]);
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kChunk = 32768;

// One thread drives the bulk engine: keep S G2S loads in flight; when stage s
// lands, issue its S2G store, and reuse the stage once the store has READ it.
__global__ void tma_copy(const char* __restrict__ a, char* __restrict__ b, size_t chunks, int S) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t first = blockIdx.x, step = gridDim.x;
  size_t issued = 0, done = 0;
  uint32_t phase[16] = {0};
  // prologue
  for (size_t c = first; c < chunks && issued < (size_t)S; c += step, ++issued) {
    const int s = issued % S;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(smem + s * kChunk)),
                 "l"(a + c * kChunk), "r"(kChunk), "r"(sa(&full[s]))
                 : "memory");
  }
  for (size_t c = first; c < chunks; c += step, ++done) {
    const int s = done % S;
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
            sa(&full[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + c * kChunk),
                 "r"(sa(smem + s * kChunk)), "r"(kChunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill stage s with chunk c + S*step once its store has been read
    const size_t cn = c + (size_t)S * step;
    if (cn < chunks) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kChunk)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(smem + s * kChunk)),
                   "l"(a + cn * kChunk), "r"(kChunk), "r"(sa(&full[s]))
                   : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = size_t(512) << 20;
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  auto time = [&](auto launch) {
    launch();
    cudaEventRecord(s);
    launch();
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    return ms;
  };
  printf("variant            sms   GB/s(r+w)  per-SM\n");
  for (int sms : {8, 16, 32, 148}) {
    const size_t nb = sms >= 32 ? bytes : bytes / 4;
    const size_t n = nb / 16;
    auto report = [&](const char* name, float ms) {
      const double gbs = 2.0 * nb / (ms * 1e-3) / 1e9;
      printf("%-18s %4d  %9.1f  %6.1f\n", name, sms, gbs, gbs / sms);
    };
    report("lsu U4 C1", time([&] { lsu_copy<4><<<sms, 1024>>>((const uint4*)a, (uint4*)b, n); }));
    report("lsu U8 C1", time([&] { lsu_copy<8><<<sms, 1024>>>((const uint4*)a, (uint4*)b, n); }));
    report("lsu U4 C2", time([&] { lsu_copy<4><<<2 * sms, 1024>>>((const uint4*)a, (uint4*)b, n); }));
    report("lsu U8 C2(512t)", time([&] { lsu_copy<8><<<4 * sms, 512>>>((const uint4*)a, (uint4*)b, n); }));
    for (int S : {2, 4, 6}) {
      char name[32];
      snprintf(name, sizeof name, "tma S%d C1", S);
      report(name, time([&] { tma_copy<<<sms, 32, S * kChunk>>>(a, b, nb / kChunk, S); }));
    }
    report("tma S3 C2", time([&] { tma_copy<<<2 * sms, 32, 3 * kChunk>>>(a, b, nb / kChunk, 3); }));
    report("tma S2 C3", time([&] { tma_copy<<<3 * sms, 32, 2 * kChunk>>>(a, b, nb / kChunk, 2); }));
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
