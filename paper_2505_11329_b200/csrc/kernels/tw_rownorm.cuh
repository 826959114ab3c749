// tw_rownorm.cuh -- the row engine shared by K1 (fused AllReduce + residual +
// RMSNorm) and K2 (TP=1 fused residual + RMSNorm).
//
// One "row group" of `tpr` threads owns one token row at a time; a CTA holds
// blockDim/tpr groups, so several rows are in flight per SM.  Per row:
//   x   = the reduced input row   (K2: local load; K1: NVLS multimem.ld_reduce
//                                  or rank-ascending sum of peer loads)
//   r'  = x + residual             (fp32; stored back rounded to the dtype)
//   ss  = sum r'^2                 (fp32 for bf16, double for fp32 -- the
//                                  reference's double accumulator,
//                                  proj/src/numerics.cpp:51-56)
//   out = r' * (1/sqrt(ss/H + eps)) * w    (proj/src/numerics.cpp:57-61)
// The row reduction is warp shuffles + a double-buffered shared partial and
// one named barrier per row (no __syncthreads on the row path).
//
// K1 brackets the row loop with the cross-rank signal-pad barrier
// (PAPER.md:418,453): CTA b of every rank adds 1 to counter b of every rank's
// pad (multimem.red on NVLS, red per peer otherwise) and waits on its own
// counter b with ld.acquire.sys for a target derived from CTA b's launch
// generation, kept in device memory (graph-replayable, no host epoch).
#pragma once

#include <cstdint>
#include <type_traits>

#include "tw_ptx.cuh"

namespace tw {

enum class Xport : int { Local = 0, Peer = 1, Nvls = 2 };

constexpr int kMaxRanks = 8;
constexpr int kMaxGroups = 16;
constexpr int kBlock = 512;  // threads per CTA upper bound (launch bounds)

struct RankSlot {
  int rank;
  int pad_;
  long long begin, end;  // owned token shard [begin, end)
  void* residual;        // shard rows [end-begin, H], updated in place
  const float* weight;   // fp32[H] on this device
  uint32_t* pad;         // this rank's signal counters, one per CTA index (unicast VA)
  uint32_t* gen;         // this rank's per-CTA-index launch generations (device-resident)
};

// Signal-pad granule of one rank: arrival counters for up to kPadSlots CTA
// indices, then each CTA index's launch generation, then the timeout flag.
// Barriers need no host-side epoch, so launches can be captured in CUDA
// graphs and replayed.
constexpr int kPadSlots = 1024;
constexpr size_t kPadGenOffset = 4096;
constexpr size_t kPadErrOffset = 8192;
constexpr size_t kPadBytes = 16384;

struct RowParams {
  long long T, H;
  long long row_offset;  // K1: first token row of the symmetric buffers this op covers
  int V;    // vectors per row (H / N)
  int tpr;  // threads per row group (multiple of 32)
  float eps;
  unsigned flags;
  // K2 (Local)
  const void* in;
  const void* res_in;
  void* res_out;
  void* out;
  const float* weight;
  // K1
  int world;
  int nslots;
  RankSlot slot[kMaxRanks];
  void* peer_in[kMaxRanks];
  void* peer_out[kMaxRanks];
  void* peer_res[kMaxRanks];
  uint32_t* peer_pad[kMaxRanks];
  void* mc_in;
  void* mc_out;
  void* mc_res;
  uint32_t* mc_pad;
  int* err;
  long long spin_limit;   // barrier poll bound before the timeout flag is raised
  int drop_arrival_rank;  // fault injection (tests): this rank never signals; -1 = none
  int nslots_stages;      // k1_peer_tma_kernel: smem ring depth
};

constexpr unsigned kGatherResidual = 0x1u;
constexpr unsigned kDeviceScope = 0x100u;  // internal: every rank on this GPU (device-scope barriers)
// internal (TW_NVLS_ALIAS_FENCE=1, A/B on an NVSwitch box): fence.proxy.alias
// before the NVLS exit arrival.  Off by default, as in the paper's kernel
// (Listing 1) and PyTorch's multimem AllReduce it builds on: the
// multicast-VA stores are read through the unicast VA only by LATER kernels.
constexpr unsigned kAliasFence = 0x200u;

// ---- typed vector access -------------------------------------------------------
// N elements of E per "vector": 8 x bf16 or 4 x f32 (16 B), or 1 element.

template <class E, int N>
struct Vec;

template <>
struct Vec<uint16_t, 8> {  // bf16 x 8
  static constexpr int kElems = 8;
  using Raw = uint4;
  static __device__ __forceinline__ Raw load(const void* base, long long e) {
    return ld_v4(static_cast<const uint16_t*>(base) + e);
  }
  static __device__ __forceinline__ Raw load_stream(const void* base, long long e) {
    return ld_stream_v4(static_cast<const uint16_t*>(base) + e);
  }
  static __device__ __forceinline__ Raw mm_reduce(const void* mc, long long e) {
    return mm_ld_reduce_bf16x8(static_cast<const uint16_t*>(mc) + e);
  }
  static __device__ __forceinline__ void store(void* base, long long e, Raw v) {
    st_v4(static_cast<uint16_t*>(base) + e, v);
  }
  static __device__ __forceinline__ void mm_store(void* mc, long long e, Raw v) {
    mm_st_v4(static_cast<uint16_t*>(mc) + e, v);
  }
  static __device__ __forceinline__ void unpack(Raw v, float (&f)[8]) {
    f[0] = bf16lo(v.x); f[1] = bf16hi(v.x); f[2] = bf16lo(v.y); f[3] = bf16hi(v.y);
    f[4] = bf16lo(v.z); f[5] = bf16hi(v.z); f[6] = bf16lo(v.w); f[7] = bf16hi(v.w);
  }
  static __device__ __forceinline__ Raw pack(const float (&f)[8]) {
    return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                      pack_bf16x2(f[6], f[7]));
  }
};

template <>
struct Vec<float, 4> {  // f32 x 4
  static constexpr int kElems = 4;
  using Raw = uint4;
  static __device__ __forceinline__ Raw load(const void* base, long long e) {
    return ld_v4(static_cast<const float*>(base) + e);
  }
  static __device__ __forceinline__ Raw load_stream(const void* base, long long e) {
    return ld_stream_v4(static_cast<const float*>(base) + e);
  }
  static __device__ __forceinline__ Raw mm_reduce(const void* mc, long long e) {
    return mm_ld_reduce_f32x4(static_cast<const float*>(mc) + e);
  }
  static __device__ __forceinline__ void store(void* base, long long e, Raw v) {
    st_v4(static_cast<float*>(base) + e, v);
  }
  static __device__ __forceinline__ void mm_store(void* mc, long long e, Raw v) {
    mm_st_v4(static_cast<float*>(mc) + e, v);
  }
  static __device__ __forceinline__ void unpack(Raw v, float (&f)[4]) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  static __device__ __forceinline__ Raw pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};

template <>
struct Vec<uint16_t, 1> {  // scalar bf16 (H not a multiple of 8)
  static constexpr int kElems = 1;
  using Raw = uint32_t;
  static __device__ __forceinline__ Raw load(const void* base, long long e) {
    return static_cast<const uint16_t*>(base)[e];
  }
  static __device__ __forceinline__ Raw load_stream(const void* base, long long e) { return load(base, e); }
  static __device__ __forceinline__ Raw mm_reduce(const void*, long long) { __trap(); return 0; }
  static __device__ __forceinline__ void store(void* base, long long e, Raw v) {
    static_cast<uint16_t*>(base)[e] = static_cast<uint16_t>(v);
  }
  static __device__ __forceinline__ void mm_store(void*, long long, Raw) { __trap(); }
  static __device__ __forceinline__ void unpack(Raw v, float (&f)[1]) { f[0] = __uint_as_float(v << 16); }
  static __device__ __forceinline__ Raw pack(const float (&f)[1]) { return f32_to_bf16(f[0]); }
};

template <>
struct Vec<float, 1> {  // scalar f32 (H not a multiple of 4)
  static constexpr int kElems = 1;
  using Raw = uint32_t;
  static __device__ __forceinline__ Raw load(const void* base, long long e) {
    return __float_as_uint(static_cast<const float*>(base)[e]);
  }
  static __device__ __forceinline__ Raw load_stream(const void* base, long long e) { return load(base, e); }
  static __device__ __forceinline__ Raw mm_reduce(const void* mc, long long e) {
    return __float_as_uint(mm_ld_reduce_f32(static_cast<const float*>(mc) + e));
  }
  static __device__ __forceinline__ void store(void* base, long long e, Raw v) {
    static_cast<float*>(base)[e] = __uint_as_float(v);
  }
  static __device__ __forceinline__ void mm_store(void* mc, long long e, Raw v) {
    mm_st_b32(static_cast<float*>(mc) + e, v);
  }
  static __device__ __forceinline__ void unpack(Raw v, float (&f)[1]) { f[0] = __uint_as_float(v); }
  static __device__ __forceinline__ Raw pack(const float (&f)[1]) { return __float_as_uint(f[0]); }
};

template <int N>
__device__ __forceinline__ void load_weight(const float* w, long long e, float (&f)[N]) {
  if constexpr (N == 8) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(w + e));
    const float4 b = __ldg(reinterpret_cast<const float4*>(w + e) + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else if constexpr (N == 4) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(w + e));
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  } else {
    f[0] = __ldg(w + e);
  }
}

template <class Acc>
__device__ __forceinline__ Acc warp_sum(Acc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// The row statistic from a row group's warp partials.  bf16 rows (Acc =
// float, 2e-2 tolerance): the partials as 16-byte loads and a tree, then one
// rsqrtf -- a chain of dependent scalar shared loads and IEEE div / sqrt /
// div sat on every row's critical path (K2's packed body: +5 % per SM under
// an SM budget).  fp32 rows (Acc = double): the reference's arithmetic,
// float(ss / H) and 1 / sqrt (proj/src/numerics.cpp:57-61), unchanged.
template <class Acc>
__device__ __forceinline__ Acc sum_partials(const Acc* parts, int n) {
  Acc t = 0;
  if constexpr (sizeof(Acc) == 4) {
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(parts) & 15) == 0) {
      for (int q = 0; q < n; q += 4) {
        const float4 v = *reinterpret_cast<const float4*>(parts + q);
        t += (v.x + v.y) + (v.z + v.w);
      }
      return t;
    }
  }
  for (int q = 0; q < n; ++q) t += parts[q];
  return t;
}

template <class Acc>
__device__ __forceinline__ float inv_rms(Acc total, long long H, float eps) {
  if constexpr (sizeof(Acc) == 4)
    return rsqrtf(total * (1.0f / static_cast<float>(H)) + eps);
  else
    return 1.0f / sqrtf(static_cast<float>(total / static_cast<Acc>(H)) + eps);
}

// ---- cross-rank barrier ------------------------------------------------------------

template <Xport X>
// phase 1 = entry, 2 = exit.  CTA b's g-th launch waits for its counter to
// reach world*(2g+phase); the exit barrier then advances the CTA's generation
// (only CTA b of this rank writes gen[b]; the next launch reads it after the
// kernel boundary).  Every rank launches the same CTA count per call, so the
// counters of CTA index b advance in lockstep across ranks.
//
// Memory semantics follow the paper's kernel (Listing 1:
// sync_remote_blocks<Relaxed> at entry, <AcqRel> at exit):
//  * entry publishes nothing this kernel wrote -- the INPUT rows were written
//    by earlier kernels, complete at the kernel boundary -- so the arrival and
//    the polls are relaxed: the barrier only says "every rank has started";
//  * exit is a release (fence, then the arrival) of this CTA's stores and an
//    acquire (relaxed polls, then one acquire load) of every peer's.
__device__ __forceinline__ void rank_barrier(const RowParams& p, const RankSlot& s, int phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int b = blockIdx.x;  // per-block-index counters: CTA b meets CTA b of every rank
    const uint32_t g = *reinterpret_cast<volatile uint32_t*>(s.gen + b);
    const uint32_t target = static_cast<uint32_t>(p.world) * (2u * g + static_cast<uint32_t>(phase));
    const bool exit = phase == 2;
    const bool dev_scope = X != Xport::Nvls && (p.flags & kDeviceScope);
    // The CTA's prior writes are ordered before the exit arrival by bar.sync
    // (cumulativity) + the release fence.
    if (s.rank != p.drop_arrival_rank) {  // fault injection: a rank that never arrives
      if constexpr (X == Xport::Nvls) {
        if (exit) {
          if (p.flags & kAliasFence) fence_proxy_alias();
          mm_red_release_add(p.mc_pad + b, 1u);  // one op reaches every rank's pad
        } else {
          mm_red_relaxed_add(p.mc_pad + b, 1u);
        }
      } else if (dev_scope) {
        if (exit) fence_acq_rel_gpu();
        for (int q = 0; q < p.world; ++q) red_relaxed_add_gpu(p.peer_pad[q] + b, 1u);
      } else {
        if (exit) fence_acq_rel_sys();
        for (int q = 0; q < p.world; ++q) red_relaxed_add(p.peer_pad[q] + b, 1u);
      }
    }
    long long spins = 0;
    while (static_cast<int>((dev_scope ? ld_relaxed_gpu(s.pad + b) : ld_relaxed_sys(s.pad + b)) - target) < 0) {
      if (++spins > p.spin_limit) {  // bounded: a rank was never launched / died
        atomicExch(p.err, 1);
        break;
      }
      // poll back to back first (a decode-size barrier completes within a few
      // us), then back off so a long wait does not flood the memory system
      if (spins > 256) __nanosleep(64);
    }
    if (exit) {
      // acquire: one ld.acquire of the counter the relaxed polls saw reach the
      // target (LDG.STRONG + CCTL.IVALL in SASS; a fence.acq_rel here would be
      // a second MEMBAR.ALL.SYS, ~3 us at system scope)
      if (dev_scope)
        (void)ld_acquire_gpu(s.pad + b);
      else
        (void)ld_acquire(s.pad + b);
      s.gen[b] = g + 1u;
    }
  }
  __syncthreads();
}

// ---- the row kernel ------------------------------------------------------------------

// PF: software-pipelined row loop (next row's loads in flight during this
// row's math and stores) -- the NVLS path, where ld_reduce latency is long;
// the local (K2) engine defaults to PF=false, which measured faster for short
// rows (TW_ROWS_PIPELINE=1 selects PF=true there, used by the tests to cover
// the pipelined code on hardware).
template <class E, int N, int VPT, Xport X, bool PF>
__global__ void __launch_bounds__(kBlock, (X == Xport::Peer && VPT <= 2) ? 2 : 1)
    rownorm_kernel(const __grid_constant__ RowParams p) {
  using VT = Vec<E, N>;
  using Raw = typename VT::Raw;
  // fp32 activations keep the reference's double sum of squares.
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  __shared__ __align__(16) Acc part[kMaxGroups][2][kBlock / 32];

  const int slot_idx = (X == Xport::Local) ? 0 : static_cast<int>(blockIdx.y);
  const RankSlot& s = p.slot[slot_idx];
  const int tpr = p.tpr;
  const int groups = blockDim.x / tpr;
  const int group = threadIdx.x / tpr;
  const int lt = threadIdx.x - group * tpr;
  const int warp_in_group = lt >> 5;
  const int nwarps = tpr >> 5;
  const long long H = p.H;

  if constexpr (X != Xport::Local) {
    rank_barrier<X>(p, s, 1);
  }

  long long row0, row1;
  if constexpr (X == Xport::Local) {
    row0 = 0;
    row1 = p.T;
  } else {
    row0 = s.begin;
    row1 = s.end;
  }
  const long long stride = static_cast<long long>(gridDim.x) * groups;
  const void* res_src = (X == Xport::Local) ? p.res_in : s.residual;
  void* res_dst = (X == Xport::Local) ? p.res_out : s.residual;
  float xs[(X == Xport::Peer) ? VPT : 1][N];  // Peer: fp32 rank-sum accumulators

  // Phase 1 of a row: issue every load of the row before using any of them.
  auto load_row = [&](long long t, Raw (&xr)[VPT], Raw (&rr)[VPT]) {
    const long long rowe = (X == Xport::Local ? t : p.row_offset + t) * H;  // row in the [T,H] buffers
    const long long srow = (X == Xport::Local) ? rowe : (t - row0) * H;  // residual row
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        const long long e = rowe + static_cast<long long>(c) * N;
        if constexpr (X == Xport::Local) {
          xr[k] = VT::load_stream(p.in, e);
        } else if constexpr (X == Xport::Nvls) {
          xr[k] = VT::mm_reduce(p.mc_in, e);
        } else {
          // Rank-ascending fp32 sum from 0.0f (proj/src/collectives.cpp:74-78).
          // Loads are issued four ranks at a time before their adds (memory-
          // level parallelism within a register budget that allows two CTAs
          // per SM); the sum itself keeps the reference's rank order.
#pragma unroll
          for (int i = 0; i < N; ++i) xs[k][i] = 0.0f;
#pragma unroll
          for (int h = 0; h < kMaxRanks; h += 4) {
            Raw raw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (h + q < p.world) raw[q] = VT::load(p.peer_in[h + q], e);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (h + q < p.world) {
                float f[N];
                VT::unpack(raw[q], f);
#pragma unroll
                for (int i = 0; i < N; ++i) xs[k][i] += f[i];
              }
            }
          }
        }
        rr[k] = VT::load_stream(res_src, srow + static_cast<long long>(c) * N);
      }
    }
  };

  // Phases 2-4 of a row, once its loads are in registers.
  auto finish_row = [&](long long t, Raw (&xr)[VPT], Raw (&rr)[VPT], int parity) {
    const long long rowe = (X == Xport::Local ? t : p.row_offset + t) * H;
    const long long srow = (X == Xport::Local) ? rowe : (t - row0) * H;
    // Phase 2: r' = x + res (fp32), rounded to the storage type and written
    // back; the sum of squares is taken over the stored (rounded) r' so the
    // output is exactly the RMSNorm of the residual the caller gets back.
    Acc ss = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        float x[N], r[N];
        if constexpr (X == Xport::Peer) {
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = xs[k][i];
        } else {
          VT::unpack(xr[k], x);
        }
        VT::unpack(rr[k], r);
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] = x[i] + r[i];
        rr[k] = VT::pack(r);
        VT::unpack(rr[k], r);
#pragma unroll
        for (int i = 0; i < N; ++i) ss += static_cast<Acc>(r[i]) * static_cast<Acc>(r[i]);
        VT::store(res_dst, srow + static_cast<long long>(c) * N, rr[k]);
        if (p.flags & kGatherResidual) {
          const long long e = rowe + static_cast<long long>(c) * N;
          if constexpr (X == Xport::Nvls) {
            VT::mm_store(p.mc_res, e, rr[k]);
          } else if constexpr (X == Xport::Peer) {
            for (int q = 0; q < p.world; ++q) VT::store(p.peer_res[q], e, rr[k]);
          }
        }
      }
    }
    // Phase 3: row reduction.
    ss = warp_sum(ss);
    Acc total;
    if (nwarps == 1) {
      total = ss;
    } else {
      if ((lt & 31) == 0) part[group][parity][warp_in_group] = ss;
      named_bar_sync(1 + group, tpr);
      total = sum_partials<Acc>(part[group][parity], nwarps);
    }
    const float inv = inv_rms<Acc>(total, H, p.eps);
    // Phase 4: out = r' * inv * w, stored locally / to every rank.
    const float* wgt = (X == Xport::Local) ? p.weight : s.weight;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        const long long e = static_cast<long long>(c) * N;
        float w[N], o[N];
        load_weight<N>(wgt, e, w);
        VT::unpack(rr[k], o);
#pragma unroll
        for (int i = 0; i < N; ++i) o[i] = o[i] * inv * w[i];
        const Raw ov = VT::pack(o);
        if constexpr (X == Xport::Local) {
          VT::store(p.out, rowe + e, ov);
        } else if constexpr (X == Xport::Nvls) {
          VT::mm_store(p.mc_out, rowe + e, ov);
        } else {
          for (int q = 0; q < p.world; ++q) VT::store(p.peer_out[q], rowe + e, ov);
        }
      }
    }
  };

  const long long first = row0 + static_cast<long long>(blockIdx.x) * groups + group;
  if constexpr (PF && X != Xport::Peer) {
    // Software pipeline: the next row's loads are in flight while this row is
    // reduced, normalised and stored (two register sets, ping-pong).
    Raw xa[VPT], ra[VPT], xb[VPT], rb[VPT];
    int parity = 0;
    long long t = first;
    if (t < row1) load_row(t, xa, ra);
    while (t < row1) {
      const long long tn = t + stride;
      if (tn < row1) load_row(tn, xb, rb);
      finish_row(t, xa, ra, parity);
      parity ^= 1;
      if (tn >= row1) break;
      const long long tnn = tn + stride;
      if (tnn < row1) load_row(tnn, xa, ra);
      finish_row(tn, xb, rb, parity);
      parity ^= 1;
      t = tnn;
    }
  } else {
    // Peer holds every rank's vector before the ordered sum: no second set.
    int parity = 0;
    for (long long t = first; t < row1; t += stride, parity ^= 1) {
      Raw xr[VPT], rr[VPT];
      load_row(t, xr, rr);
      finish_row(t, xr, rr, parity);
    }
  }

  if constexpr (X != Xport::Local) rank_barrier<X>(p, s, 2);
}

}  // namespace tw
