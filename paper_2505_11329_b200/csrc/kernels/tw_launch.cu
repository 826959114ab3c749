// tw_launch.cu -- instantiation and launch of the row engine (K1, K2) and of
// the unfused AllReduce baseline kernel (K3).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "tw_bulk.cuh"
#include "tw_flat.cuh"
#include "tw_launch.h"
#include "tw_rownorm.cuh"

namespace tw {

// ---- per-function launch setup, cached ---------------------------------------------
// cudaFuncSetAttribute and the occupancy calculator cost microseconds of host
// time per call; at decode sizes that is the whole op.  Both are per (function,
// device) facts, so they are computed once (tools/host_overhead.py).
namespace {
std::mutex g_setup_mu;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

cudaError_t ensure_dynamic_smem(const void* fn, size_t bytes) {
  static std::map<std::pair<const void*, int>, size_t> set;
  const auto key = std::make_pair(fn, current_device());
  std::lock_guard<std::mutex> g(g_setup_mu);
  auto it = set.find(key);
  if (it != set.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) set[key] = bytes;
  return e;
}

int cached_occupancy(const void* fn, int threads, size_t smem) {
  static std::map<std::tuple<const void*, int, int, size_t>, int> occ;
  const auto key = std::make_tuple(fn, current_device(), threads, smem);
  {
    std::lock_guard<std::mutex> g(g_setup_mu);
    auto it = occ.find(key);
    if (it != occ.end()) return it->second;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> g(g_setup_mu);
  occ[key] = n;
  return n;
}

// ---- K3: one-shot AllReduce baseline (collectives.cpp:82-88 semantics) --------
// Rank r reduces its token shard and broadcasts it: OUTPUT[t] = sum_q INPUT_q[t].
template <class E, int N, Xport X>
__global__ void __launch_bounds__(kBlock, 1) allreduce_kernel(const __grid_constant__ RowParams p) {
  using VT = Vec<E, N>;
  const RankSlot& s = p.slot[blockIdx.y];
  rank_barrier<X>(p, s, 1);
  const long long n = (s.end - s.begin) * p.V;  // vectors in the shard
  const long long base = (p.row_offset + s.begin) * p.H;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  if constexpr (X == Xport::Nvls) {
    for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
      const long long e = base + v * N;
      VT::mm_store(p.mc_out, e, VT::mm_reduce(p.mc_in, e));
    }
  } else {
    // U vectors per thread per pass and the peers' loads issued four at a
    // time before they are summed (a load-then-add loop over the ranks kept
    // ~one load in flight per thread: the baseline ran at ~50 % of HBM).  The
    // sum stays rank-ascending fp32 from 0 (reduce_element,
    // collectives.cpp:74-78), so results are unchanged bit for bit.
    constexpr int U = 2;
    for (long long v0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v0 < n; v0 += U * stride) {
      float acc[U][N];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < N; ++i) acc[u][i] = 0.0f;
#pragma unroll
      for (int h = 0; h < kMaxRanks; h += 4) {
        if (h >= p.world) break;
        typename VT::Raw raw[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (h + q < p.world && v0 + u * stride < n) raw[u][q] = VT::load(p.peer_in[h + q], base + (v0 + u * stride) * N);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (h + q < p.world && v0 + u * stride < n) {
              float f[N];
              VT::unpack(raw[u][q], f);
#pragma unroll
              for (int i = 0; i < N; ++i) acc[u][i] += f[i];
            }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v0 + u * stride >= n) continue;
        const auto packed = VT::pack(acc[u]);
        const long long e = base + (v0 + u * stride) * N;
        for (int q = 0; q < p.world; ++q) VT::store(p.peer_out[q], e, packed);
      }
    }
  }
  rank_barrier<X>(p, s, 2);
}

namespace {

using KernelFn = void (*)(RowParams);

template <class E, int N, Xport X, bool PF>
KernelFn pick_rownorm(int vpt) {
  switch (vpt) {
    case 1: return rownorm_kernel<E, N, 1, X, PF>;
    case 2: return rownorm_kernel<E, N, 2, X, PF>;
    case 4: return rownorm_kernel<E, N, 4, X, PF>;
    case 8: return rownorm_kernel<E, N, 8, X, PF>;
    case 16: return rownorm_kernel<E, N, 16, X, PF>;
    default: return nullptr;
  }
}

// NVLS always runs the software-pipelined loop; PEER never (it already holds
// every rank's vector); the local engine runs it on request (plan.pipeline).
template <class E, int N>
KernelFn pick_by_xport(Xport x, int vpt, bool pipeline) {
  switch (x) {
    case Xport::Local:
      return pipeline ? pick_rownorm<E, N, Xport::Local, true>(vpt) : pick_rownorm<E, N, Xport::Local, false>(vpt);
    case Xport::Peer: return pick_rownorm<E, N, Xport::Peer, false>(vpt);
    case Xport::Nvls: return nullptr;  // k1_nvls_kernel (tw_nvls.cuh)
  }
  return nullptr;
}

KernelFn pick_kernel(bool bf16, int N, Xport x, int vpt, bool pipeline) {
  if (bf16)
    return N == 8 ? pick_by_xport<uint16_t, 8>(x, vpt, pipeline) : pick_by_xport<uint16_t, 1>(x, vpt, pipeline);
  return N == 4 ? pick_by_xport<float, 4>(x, vpt, pipeline) : pick_by_xport<float, 1>(x, vpt, pipeline);
}

KernelFn pick_allreduce(bool bf16, int N, Xport x) {
  if (x == Xport::Nvls) return nullptr;  // k3_nvls_kernel (tw_nvls.cuh)
  if (bf16) return N == 8 ? allreduce_kernel<uint16_t, 8, Xport::Peer> : allreduce_kernel<uint16_t, 1, Xport::Peer>;
  return N == 4 ? allreduce_kernel<float, 4, Xport::Peer> : allreduce_kernel<float, 1, Xport::Peer>;
}

int round32(long long x) { return static_cast<int>(((x + 31) / 32) * 32); }

}  // namespace

bool plan_rows(long long H, int elems_per_vec, int tpr_pref, RowPlan* plan) {
  if (H < 1 || H % elems_per_vec) return false;
  const long long V = H / elems_per_vec;
  const int vpts[] = {1, 2, 4, 8, 16};
  for (int vpt : vpts) {
    const int tpr = std::max(32, round32((V + vpt - 1) / vpt));
    if (tpr <= tpr_pref || (vpt == 16 && tpr <= kBlock)) {
      plan->N = elems_per_vec;
      plan->V = static_cast<int>(V);
      plan->vpt = vpt;
      plan->tpr = tpr;
      plan->groups = std::min(kMaxGroups, kBlock / tpr);
      plan->pipeline = false;
      return true;
    }
  }
  return false;
}

cudaError_t launch_rownorm(const RowParams& params, const RowPlan& plan, bool bf16, Xport x, dim3 grid,
                           cudaStream_t stream) {
  KernelFn fn = pick_kernel(bf16, plan.N, x, plan.vpt, plan.pipeline);
  if (!fn) return cudaErrorInvalidConfiguration;
  RowParams p = params;
  p.V = plan.V;
  p.tpr = plan.tpr;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, dim3(plan.groups * plan.tpr), args, 0, stream);
}

cudaError_t launch_allreduce(const RowParams& params, const RowPlan& plan, bool bf16, Xport x, dim3 grid,
                             cudaStream_t stream) {
  KernelFn fn = pick_allreduce(bf16, plan.N, x);
  if (!fn) return cudaErrorInvalidConfiguration;
  RowParams p = params;
  p.V = plan.V;
  p.tpr = plan.tpr;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, dim3(kBlock), args, 0, stream);
}

int rownorm_blocks_per_sm(const RowPlan& plan, bool bf16, Xport x) {
  KernelFn fn = pick_kernel(bf16, plan.N, x, plan.vpt, plan.pipeline);
  if (!fn) return 0;
  return cached_occupancy(reinterpret_cast<const void*>(fn), plan.groups * plan.tpr, 0);
}

// ---- K2 bulk-copy pipeline -------------------------------------------------------

namespace {
using BulkFn = void (*)(BulkParams);

template <class E, int G>
BulkFn pick_bulk_eg(int vpt, bool tma_store) {
  switch (vpt) {
    case 1: return tma_store ? k2_tma_kernel<E, 1, G> : k2_bulk_kernel<E, 1>;
    case 2: return tma_store ? k2_tma_kernel<E, 2, G> : k2_bulk_kernel<E, 2>;
    case 4: return tma_store ? k2_tma_kernel<E, 4, G> : k2_bulk_kernel<E, 4>;
    case 8: return tma_store ? k2_tma_kernel<E, 8, G> : k2_bulk_kernel<E, 8>;
    default: return nullptr;
  }
}

template <class E>
BulkFn pick_bulk_e(int vpt, bool tma_store, int groups) {
  return groups == 2 ? pick_bulk_eg<E, 2>(vpt, tma_store) : pick_bulk_eg<E, 1>(vpt, tma_store);
}
}  // namespace

size_t bulk_smem_bytes(int stages, uint32_t row_bytes, int tpr, int groups) {
  return static_cast<size_t>(stages) * 2 * row_bytes + 2 * stages * sizeof(uint64_t) +
         2 * static_cast<size_t>(std::max(groups, 1)) * (tpr / 32) * sizeof(double);
}

cudaError_t launch_k2_bulk(const BulkParams& params, int vpt, bool bf16, int grid, cudaStream_t stream,
                           bool tma_store) {
  BulkParams p = params;
  if (!tma_store || p.groups != 2) p.groups = 1;  // the register-store engine has one row group
  BulkFn fn = bf16 ? pick_bulk_e<uint16_t>(vpt, tma_store, p.groups) : pick_bulk_e<float>(vpt, tma_store, p.groups);
  if (!fn) return cudaErrorInvalidConfiguration;
  const size_t smem = bulk_smem_bytes(p.stages, p.row_bytes, p.tpr, p.groups);
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(p.groups * p.tpr + 32), args, smem,
                          stream);
}

// ---- K2 flat engine ----------------------------------------------------------------

cudaError_t launch_k2_flat(const FlatParams& params, bool bf16, int sms, bool one_cta_per_sm, cudaStream_t stream) {
  const int vpt_needed = (params.V + 1023) / 1024;
  using FlatFn = void (*)(FlatParams);
  FlatFn fn = nullptr;
  int vpt = 0;
  if (vpt_needed <= 1) {
    fn = bf16 ? k2_flat_kernel<uint16_t, 1> : k2_flat_kernel<float, 1>;
    vpt = 1;
  } else if (vpt_needed <= 2) {
    fn = bf16 ? k2_flat_kernel<uint16_t, 2> : k2_flat_kernel<float, 2>;
    vpt = 2;
  } else {
    return cudaErrorInvalidConfiguration;
  }
  const int threads = std::max(32, ((params.V + vpt - 1) / vpt + 31) / 32 * 32);
  int per_sm = one_cta_per_sm ? 1 : cached_occupancy(reinterpret_cast<const void*>(fn), threads, 0);
  if (one_cta_per_sm) per_sm = 1;  // an explicit SM budget: more CTAs would spread over more SMs
  const long long grid = std::min<long long>(params.T, static_cast<long long>(sms) * std::max(per_sm, 1));
  FlatParams p = params;
  void* args[] = {&p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(static_cast<unsigned>(grid)), dim3(threads), args,
                          0, stream);
}

// ---- finite scan (TokenMatrix::validate, numerics.cpp:25-27) ---------------------

template <class E>
__global__ void count_nonfinite_kernel(const E* x, long long n, int* count) {
  int local = 0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float f;
    if constexpr (sizeof(E) == 2) {
      f = bf16_to_f32(x[i]);
    } else {
      f = x[i];
    }
    local += !isfinite(f);
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

cudaError_t launch_count_nonfinite(const void* x, long long n, bool bf16, int* count, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int block = 256;
  const int grid = static_cast<int>(std::min<long long>((n + block - 1) / block, 148LL * 8));
  if (bf16)
    count_nonfinite_kernel<uint16_t><<<grid, block, 0, stream>>>(static_cast<const uint16_t*>(x), n, count);
  else
    count_nonfinite_kernel<float><<<grid, block, 0, stream>>>(static_cast<const float*>(x), n, count);
  return cudaGetLastError();
}

// ---- K1 over PEER as a bulk-copy pipeline ---------------------------------------------

namespace {
using PeerTmaFn = void (*)(RowParams);

template <class E, int W, int G = 1>
PeerTmaFn pick_peer_tma_w(int vpt) {
  vpt = vpt <= 1 ? 1 : vpt <= 2 ? 2 : vpt <= 4 ? 4 : 0;  // c < V guards the rest
  switch (vpt) {
    case 1: return k1_peer_tma_kernel<E, 1, W, G>;
    case 2: return k1_peer_tma_kernel<E, 2, W, G>;
    case 4: return k1_peer_tma_kernel<E, 4, W, G>;
    default: return nullptr;
  }
}

// Consumer row groups of the PEER engine.  Two groups (two rows in flight
// per CTA) pay at world 2 -- co-located TP=2, bf16, T=8192, 8 SMs: H=8192
// 635 -> 553 us, H=4096 473 -> 344 us; never slower beyond noise at larger
// budgets -- while world 3 loses its third stage to the even-ring rule
// (S=2) and is slower (profiles/k2_packed_ab_r02.txt section 16).
// TW_K1_PEER_GROUPS=1|2 forces the choice (world <= 3).
int peer_tma_groups(int world, int /*blocks*/) {
  static const char* env = std::getenv("TW_K1_PEER_GROUPS");
  if (world > 3) return 1;
  if (env && (env[0] == '1' || env[0] == '2')) return env[0] - '0';
  return world == 2 ? 2 : 1;
}

// Worlds 2, 3, 4 (one stage per row) and 8 (two); others use the row engine.
template <class E>
PeerTmaFn pick_peer_tma(int world, int vpt, int G) {
  switch (world) {
    case 2: return G == 2 ? pick_peer_tma_w<E, 2, 2>(vpt) : pick_peer_tma_w<E, 2>(vpt);
    case 3: return G == 2 ? pick_peer_tma_w<E, 3, 2>(vpt) : pick_peer_tma_w<E, 3>(vpt);
    case 4: return pick_peer_tma_w<E, 4>(vpt);
    case 8: return pick_peer_tma_w<E, 8>(vpt);
    default: return nullptr;
  }
}

// Ring depth under a 200 KB shared-memory budget: peer_tma_stage_rows(W)
// rows per stage, 2..4 stages, a multiple of the row groups (0 = the shape
// does not fit).
bool peer_tma_geometry(int world, int G, long long H, bool bf16, int* stages, size_t* smem) {
  const size_t row = static_cast<size_t>(H) * (bf16 ? 2 : 4);
  const size_t stage = peer_tma_stage_rows(world) * row;
  static const char* env = std::getenv("TW_K1_PEER_STAGES");  // A/B: ring depth cap
  const int cap = env ? std::max(2, std::atoi(env)) : 4;
  int S = static_cast<int>(std::min<size_t>(cap, (200 * 1024) / stage));
  S -= S % G;  // each row group's stages are its own (k1_peer_tma_kernel)
  if (S < 2) return false;
  *stages = S;
  *smem = S * stage + 2 * S * sizeof(uint64_t) + G * 2 * 8 * sizeof(double);
  return true;
}
}  // namespace

// Resident CTAs per SM of the engine a launch may pick: the minimum over the
// one- and two-group kernels (the grid is sized before the group count is
// chosen, and co-located ranks need every CTA resident for the rank barrier).
int k1_peer_tma_blocks_per_sm(int world, int V, long long H, bool bf16) {
  const int vpt = (V + 255) / 256;
  int occ = 0;
  for (int G = 1; G <= (world <= 3 ? 2 : 1); ++G) {
    PeerTmaFn fn = bf16 ? pick_peer_tma<uint16_t>(world, vpt, G) : pick_peer_tma<float>(world, vpt, G);
    int S = 0;
    size_t smem = 0;
    if (!fn || !peer_tma_geometry(world, G, H, bf16, &S, &smem)) {
      if (G == 1) return 0;
      continue;  // the launcher falls back to one group
    }
    if (ensure_dynamic_smem(reinterpret_cast<const void*>(fn), smem) != cudaSuccess) return 0;
    const int o = cached_occupancy(reinterpret_cast<const void*>(fn), G * 256 + 32, smem);
    occ = G == 1 ? o : std::min(occ, o);
  }
  return occ;
}

cudaError_t launch_k1_peer_tma(RowParams params, int world, int V, bool bf16, dim3 grid, cudaStream_t stream) {
  const int vpt = (V + 255) / 256;
  int G = peer_tma_groups(world, static_cast<int>(grid.x));
  int S = 0;
  size_t smem = 0;
  if (G > 1 && !peer_tma_geometry(world, G, params.H, bf16, &S, &smem)) G = 1;
  PeerTmaFn fn = bf16 ? pick_peer_tma<uint16_t>(world, vpt, G) : pick_peer_tma<float>(world, vpt, G);
  if (!fn || !peer_tma_geometry(world, G, params.H, bf16, &S, &smem)) return cudaErrorNotSupported;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  params.V = V;
  params.nslots_stages = S;
  params.world = world;
  void* args[] = {&params};
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), grid, dim3(G * 256 + 32), args, smem, stream);
}

}  // namespace tw
