// tw_nvls.cu -- instantiation and launch of the NVLS kernels (tw_nvls.cuh):
// K1 (fused AllReduce + residual + RMSNorm) and the K3 AllReduce baseline,
// each for the hardware multimem policy and the co-located simulation.
#include <cuda_runtime.h>

#include "tw_launch.h"
#include "tw_nvls.cuh"

namespace tw {

// ---- K1 / K3 over NVLS (tw_nvls.cuh) ---------------------------------------------------

namespace {
using KernelFn = void (*)(RowParams);

template <class E, int D, class MM>
KernelFn pick_nvls_d(int vpt) {
  switch (vpt) {
    case 1: return k1_nvls_kernel<E, 1, D, MM>;
    case 2: return k1_nvls_kernel<E, 2, D, MM>;
    case 4: return k1_nvls_kernel<E, 4, D, MM>;
    default: return nullptr;
  }
}

template <class E, class MM>
KernelFn pick_nvls_e(int vpt, int depth) {
  switch (depth) {
    case 1: return pick_nvls_d<E, 1, MM>(vpt);
    case 2: return pick_nvls_d<E, 2, MM>(vpt);
    case 3: return pick_nvls_d<E, 3, MM>(vpt);
    default: return nullptr;
  }
}

KernelFn pick_nvls(bool bf16, bool sim, int vpt, int depth) {
  if (bf16) return sim ? pick_nvls_e<uint16_t, MmSim>(vpt, depth) : pick_nvls_e<uint16_t, MmHw>(vpt, depth);
  return sim ? pick_nvls_e<float, MmSim>(vpt, depth) : pick_nvls_e<float, MmHw>(vpt, depth);
}
}  // namespace

int nvls_depth_from_flags(unsigned flags) {
  const int d = static_cast<int>((flags & kNvlsDepthMask) >> kNvlsDepthShift);
  return d == 0 ? kNvlsDefaultDepth : d;
}

// <= 4 vectors per thread: the D + 1 in-flight register sets stay spill-free
// (bf16 H <= 16384, fp32 H <= 8192).
bool nvls_supported(const RowPlan& plan) { return plan.vpt <= 4 && plan.groups * plan.tpr <= kNvlsBlock; }

cudaError_t launch_k1_nvls(const RowParams& params, const RowPlan& plan, bool bf16, bool sim, int depth, dim3 grid,
                           cudaStream_t stream) {
  KernelFn fn = pick_nvls(bf16, sim, plan.vpt, depth);
  if (!fn) return cudaErrorInvalidConfiguration;
  RowParams p = params;
  p.V = plan.V;
  p.tpr = plan.tpr;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, dim3(plan.groups * plan.tpr), args, 0, stream);
}

int k1_nvls_blocks_per_sm(const RowPlan& plan, bool bf16, bool sim, int depth) {
  KernelFn fn = pick_nvls(bf16, sim, plan.vpt, depth);
  if (!fn) return 0;
  return cached_occupancy(reinterpret_cast<const void*>(fn), plan.groups * plan.tpr, 0);
}

cudaError_t launch_k3_nvls(const RowParams& params, const RowPlan& plan, bool bf16, bool sim, dim3 grid,
                           cudaStream_t stream) {
  KernelFn fn = nullptr;
  if (bf16 && plan.N == 8) fn = sim ? k3_nvls_kernel<uint16_t, MmSim> : k3_nvls_kernel<uint16_t, MmHw>;
  if (!bf16 && plan.N == 4) fn = sim ? k3_nvls_kernel<float, MmSim> : k3_nvls_kernel<float, MmHw>;
  if (!fn) return cudaErrorInvalidConfiguration;
  RowParams p = params;
  p.V = plan.V;
  p.tpr = plan.tpr;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, dim3(kNvlsBlock), args, 0, stream);
}

}  // namespace tw
