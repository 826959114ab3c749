// tw_nvls.cuh -- K1 over NVLS: the north_star kernel.
//
//   reduce-scatter   x  = multimem.ld_reduce(INPUT[t])  for t in this rank's shard
//   residual + norm  r' = x + res;  out = r' * rsqrt(mean(r'^2) + eps) * w
//   all-gather       multimem.st(OUTPUT[t], out)  (+ multimem.st(RESIDUAL[t], r') with G = 2)
//
// bracketed by signal-pad barriers (Listing 1; semantics of
// proj/src/collectives.cpp:134-182).  One CTA per SM, `sm_budget` CTAs per
// rank; a CTA holds groups of `tpr` threads and a group owns whole token rows
// (the row reduction stays on chip: warp shuffles + one named barrier).
//
// Latency hiding.  An ld_reduce is a round trip through the NVSwitch to every
// rank's HBM, several times an HBM load's latency, and RMSNorm needs the whole
// row before anything can be stored.  Each group therefore keeps the
// ld_reduce of the next D rows in flight (D = 1..3, a per-call knob) while it
// normalises and multicasts the current one; the local residual row is loaded
// one row ahead.  In flight per SM at D = 2, H = 8192 bf16: 2 groups x 2 rows
// x 16 KB = 64 KB of reductions (SURVEY §7.4-1 estimates ~20-60 KB are needed
// per SM at <= 8 SMs: each SM moves only S/(N*SMs) of reductions).  The
// weights are re-read from L1 per row (32 KB fp32 per row at H = 8192), so the
// registers go to in-flight rows.
//
// The multimem operations are a policy (MM):
//   MmHw   multimem.ld_reduce / multimem.st / multimem.red on the multicast
//          VA (one rank per GPU; what an NVSwitch box runs);
//   MmSim  the same operations spelled as per-rank loads / stores / reds on
//          co-located ranks (TW_TRANSPORT_NVLS_SIM; a test transport for one
//          GPU: rank-ascending fp32 sum then one rounding, which is what
//          .acc::f32 computes up to the switch's summation order).
// Everything else -- row partition, the pipeline, barrier phases and
// generations, G = 2, fences -- is the same instantiated code, so the one-GPU
// parity/soak/graph tests exercise the NVLS kernel's whole control flow; only
// the three multimem instructions need an NVSwitch.
//
// Memory ordering (PTX ISA memory model; see DESIGN.md §7 "NVLS ordering"):
// INPUT is written by the producer through the unicast VA (an earlier kernel)
// and read by peers' ld_reduce through the multicast VA; OUTPUT/RESIDUAL are
// written through the multicast VA and read by later kernels through the
// unicast VA.  As in the paper's kernel (Listing 1:
// sync_remote_blocks<Relaxed> at entry, <AcqRel> at exit):
//  * entry: relaxed arrival + relaxed polls -- what it guards was written
//    before this kernel started (complete at the kernel boundary);
//  * exit: multimem.red.release.sys (MEMBAR.ALL.SYS + the reduction,
//    cumulative over the CTA's stores via bar.sync), relaxed polls of the
//    local pad, then one ld.acquire.sys of it (LDG.STRONG.SYS + CCTL.IVALL).
// The cross-alias reads happen only in later kernels, so no fence.proxy.alias
// is issued by default (TW_NVLS_ALIAS_FENCE=1 adds one before the exit
// arrival: MEMBAR.SC.GPU + MEMBAR.SC.SYS + CCTL.IVALL, for A/B on hardware).
// Each barrier thus costs one system-scope MEMBAR per CTA (the release).
#pragma once

#include <cstdint>
#include <type_traits>

#include "tw_ptx.cuh"
#include "tw_rownorm.cuh"

namespace tw {

constexpr int kNvlsBlock = 512;
constexpr int kNvlsMaxDepth = 3;

// Pipeline depth from the fused op's flags (TW_NVLS_DEPTH(d), 0 = default).
constexpr unsigned kNvlsDepthShift = 4;
constexpr unsigned kNvlsDepthMask = 0x3u << kNvlsDepthShift;
constexpr int kNvlsDefaultDepth = 2;

struct MmHw {
  static constexpr bool kSim = false;
  template <class VT>
  static __device__ __forceinline__ typename VT::Raw reduce(const RowParams& p, long long e) {
    return VT::mm_reduce(p.mc_in, e);
  }
  template <class VT>
  static __device__ __forceinline__ void store_out(const RowParams& p, long long e, typename VT::Raw v) {
    VT::mm_store(p.mc_out, e, v);
  }
  template <class VT>
  static __device__ __forceinline__ void store_res(const RowParams& p, long long e, typename VT::Raw v) {
    VT::mm_store(p.mc_res, e, v);
  }
  // One reduction on the multicast pad reaches counter b of every rank:
  // release at exit, relaxed at entry (see nvls_barrier).
  static __device__ __forceinline__ void arrive(const RowParams& p, int b, bool exit) {
    if (exit)
      mm_red_release_add(p.mc_pad + b, 1u);
    else
      mm_red_relaxed_add(p.mc_pad + b, 1u);
  }
  static __device__ __forceinline__ uint32_t poll(const uint32_t* pad) { return ld_relaxed_sys(pad); }
  static __device__ __forceinline__ void acquire(const uint32_t* pad) { (void)ld_acquire(pad); }
};

struct MmSim {
  static constexpr bool kSim = true;
  template <class VT>
  static __device__ __forceinline__ typename VT::Raw reduce(const RowParams& p, long long e) {
    float acc[VT::kElems];
#pragma unroll
    for (int i = 0; i < VT::kElems; ++i) acc[i] = 0.0f;
#pragma unroll
    for (int h = 0; h < kMaxRanks; h += 4) {
      typename VT::Raw raw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (h + q < p.world) raw[q] = VT::load(p.peer_in[h + q], e);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (h + q < p.world) {
          float f[VT::kElems];
          VT::unpack(raw[q], f);
#pragma unroll
          for (int i = 0; i < VT::kElems; ++i) acc[i] += f[i];
        }
      }
    }
    return VT::pack(acc);
  }
  template <class VT>
  static __device__ __forceinline__ void store_out(const RowParams& p, long long e, typename VT::Raw v) {
    for (int q = 0; q < p.world; ++q) VT::store(p.peer_out[q], e, v);
  }
  template <class VT>
  static __device__ __forceinline__ void store_res(const RowParams& p, long long e, typename VT::Raw v) {
    for (int q = 0; q < p.world; ++q) VT::store(p.peer_res[q], e, v);
  }
  // Co-located ranks share one GPU: device scope is the multicast's analogue.
  static __device__ __forceinline__ void arrive(const RowParams& p, int b, bool exit) {
    if (exit) fence_acq_rel_gpu();
    for (int q = 0; q < p.world; ++q) red_relaxed_add_gpu(p.peer_pad[q] + b, 1u);
  }
  static __device__ __forceinline__ uint32_t poll(const uint32_t* pad) { return ld_relaxed_gpu(pad); }
  static __device__ __forceinline__ void acquire(const uint32_t* pad) { (void)ld_acquire_gpu(pad); }
};

// phase 1 = entry, 2 = exit.  CTA b's g-th launch waits for its counter to
// reach world * (2g + phase); the exit barrier advances the CTA's generation
// (device-resident, so launches are graph-replayable without a host epoch).
// Semantics as PAPER.md Listing 1 (sync_remote_blocks<Relaxed> at entry,
// <AcqRel> at exit): the entry barrier publishes nothing this kernel wrote
// (INPUT was written by earlier kernels, complete at the kernel boundary), so
// it is a relaxed arrival + relaxed polls; the exit barrier releases this
// CTA's multicast stores and acquires the peers'.
template <class MM>
__device__ __forceinline__ void nvls_barrier(const RowParams& p, const RankSlot& s, int phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int b = blockIdx.x;
    const bool exit = phase == 2;
    const uint32_t g = *reinterpret_cast<volatile uint32_t*>(s.gen + b);
    const uint32_t target = static_cast<uint32_t>(p.world) * (2u * g + static_cast<uint32_t>(phase));
    // exit: this CTA's multicast-VA stores (OUTPUT, RESIDUAL) are read
    // through the unicast VA by later kernels; an optional proxy fence on the
    // writer side (kAliasFence, off by default -- see tw_rownorm.cuh).
    if (exit && (p.flags & kAliasFence)) fence_proxy_alias();
    if (s.rank != p.drop_arrival_rank) MM::arrive(p, b, exit);  // fault injection: a rank that never arrives
    long long spins = 0;
    while (static_cast<int>(MM::poll(s.pad + b) - target) < 0) {
      if (++spins > p.spin_limit) {  // bounded: a rank was never launched / died
        atomicExch(p.err, 1);
        break;
      }
      __nanosleep(32);
    }
    if (exit) {
      MM::acquire(s.pad + b);  // one acquire load (no second MEMBAR.SYS)
      s.gen[b] = g + 1u;
    }
  }
  __syncthreads();
}

// E: element type (uint16_t = bf16 bits, float).  VPT: 16-byte vectors per
// thread per row.  D: rows of ld_reduce in flight ahead of the current one.
template <class E, int VPT, int D, class MM>
__global__ void __launch_bounds__(kNvlsBlock, 1) k1_nvls_kernel(const __grid_constant__ RowParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Raw = typename VT::Raw;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;  // reference: double ss for fp32
  constexpr int kSets = D + 1;                           // x register sets (ring)
  constexpr int U = (kSets % 2 == 0) ? kSets : 2 * kSets;  // unroll: x ring and residual ping-pong align
  __shared__ __align__(16) Acc part[kMaxGroups][2][kNvlsBlock / 32];

  const RankSlot& s = p.slot[MM::kSim ? blockIdx.y : 0];
  const int tpr = p.tpr;
  const int groups = blockDim.x / tpr;
  const int group = threadIdx.x / tpr;
  const int lt = threadIdx.x - group * tpr;
  const int nwarps = tpr >> 5;
  const long long H = p.H;

  nvls_barrier<MM>(p, s, 1);

  const long long row0 = s.begin, row1 = s.end;
  const long long stride = static_cast<long long>(gridDim.x) * groups;
  const long long first = row0 + static_cast<long long>(blockIdx.x) * groups + group;
  const long long nrows = first < row1 ? (row1 - 1 - first) / stride + 1 : 0;

  auto row_of = [&](long long i) { return first + i * stride; };
  auto load_x = [&](long long t, Raw (&xr)[VPT]) {
    const long long rowe = (p.row_offset + t) * H;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) xr[k] = MM::template reduce<VT>(p, rowe + static_cast<long long>(c) * N);
    }
  };
  auto load_r = [&](long long t, Raw (&rr)[VPT]) {
    const long long srow = (t - row0) * H;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) rr[k] = VT::load_stream(s.residual, srow + static_cast<long long>(c) * N);
    }
  };
  auto finish = [&](long long t, Raw (&xr)[VPT], Raw (&rr)[VPT], int parity) {
    const long long rowe = (p.row_offset + t) * H;
    const long long srow = (t - row0) * H;
    Acc ss = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        float x[N], r[N];
        VT::unpack(xr[k], x);
        VT::unpack(rr[k], r);
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] = x[i] + r[i];
        rr[k] = VT::pack(r);  // r' rounded to the storage type; ss and out use the rounded value
        VT::unpack(rr[k], r);
#pragma unroll
        for (int i = 0; i < N; ++i) ss += static_cast<Acc>(r[i]) * static_cast<Acc>(r[i]);
        const long long ce = static_cast<long long>(c) * N;
        VT::store(s.residual, srow + ce, rr[k]);
        if (p.flags & kGatherResidual) MM::template store_res<VT>(p, rowe + ce, rr[k]);
      }
    }
    ss = warp_sum(ss);
    Acc total;
    if (nwarps == 1) {
      total = ss;
    } else {
      if ((lt & 31) == 0) part[group][parity][lt >> 5] = ss;
      named_bar_sync(1 + group, tpr);
      total = sum_partials<Acc>(part[group][parity], nwarps);
    }
    const float inv = inv_rms<Acc>(total, H, p.eps);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        const long long ce = static_cast<long long>(c) * N;
        float w[N], o[N];
        load_weight<N>(s.weight, ce, w);
        VT::unpack(rr[k], o);
#pragma unroll
        for (int i = 0; i < N; ++i) o[i] = o[i] * inv * w[i];
        MM::template store_out<VT>(p, rowe + ce, VT::pack(o));
      }
    }
  };

  Raw xq[kSets][VPT];
  Raw rq[2][VPT];
#pragma unroll
  for (int j = 0; j < D; ++j)
    if (j < nrows) load_x(row_of(j), xq[j]);
  if (nrows > 0) load_r(row_of(0), rq[0]);
  for (long long base = 0; base < nrows; base += U) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long i = base + j;
      if (i < nrows) {
        if (i + D < nrows) load_x(row_of(i + D), xq[(j + D) % kSets]);
        if (i + 1 < nrows) load_r(row_of(i + 1), rq[(j + 1) % 2]);
        finish(row_of(i), xq[j % kSets], rq[j % 2], static_cast<int>(i & 1));
      }
    }
  }

  nvls_barrier<MM>(p, s, 2);
}

// K3 (unfused AllReduce baseline) over NVLS: OUTPUT[t] = sum_r INPUT_r[t] for
// the rank's shard, multicast to every rank (collectives.cpp:82-88 semantics).
template <class E, class MM>
__global__ void __launch_bounds__(kNvlsBlock, 1) k3_nvls_kernel(const __grid_constant__ RowParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  const RankSlot& s = p.slot[MM::kSim ? blockIdx.y : 0];
  nvls_barrier<MM>(p, s, 1);
  const long long n = (s.end - s.begin) * p.V;
  const long long base = (p.row_offset + s.begin) * p.H;
  for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = base + v * N;
    MM::template store_out<VT>(p, e, MM::template reduce<VT>(p, e));
  }
  nvls_barrier<MM>(p, s, 2);
}

}  // namespace tw
