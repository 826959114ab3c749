// tw_bulk.cuh -- K2 (TP=1 fused residual-add + RMSNorm) as a warp-specialised
// bulk-copy pipeline for sm_100a.
//
// Persistent grid, one CTA per SM.  Warp 0 lane 0 is the producer: for each
// row it owns it arms a full-barrier with the row's byte count and issues two
// cp.async.bulk (TMA bulk engine) copies, input row and residual row, into a
// ring of S shared-memory stages (S*2*row_bytes <= ~200 KB).  The remaining
// warps are consumers: wait on the stage's full barrier, read the row from
// shared memory, r' = x + res (stored to global as soon as it is formed), hand
// the stage back (empty barrier), reduce the sum of squares across the
// consumer warps (one named barrier), and store out = r' * inv_rms * w with w
// held in registers for the whole kernel.  HBM traffic is exactly the
// algorithmic 4*T*H*elem bytes; up to S rows per SM are in flight.
#pragma once

#include <cstdint>

#include "tw_ptx.cuh"
#include "tw_rownorm.cuh"

namespace tw {

// Per-CTA event timestamps for tools/probe/k2trace.cu (never defined in the product build).
#ifdef TW_K2_TRACE
__device__ unsigned long long k2_trace[1024 * 64];
__device__ __forceinline__ void k2_tr(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (slot < 64) k2_trace[blockIdx.x * 64 + slot] = t;
}
// k2_tr after `dep` has been computed (the empty asm consumes it first).
__device__ __forceinline__ void k2_tr_after(int slot, float dep) {
  asm volatile("" ::"f"(dep));
  k2_tr(slot);
}
#else
__device__ __forceinline__ void k2_tr(int) {}
__device__ __forceinline__ void k2_tr_after(int, float) {}
#endif

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Global -> shared bulk copy completing on an mbarrier (TMA bulk engine).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint4 lds_v4(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_addr(p)));
  return v;
}

struct BulkParams {
  const void* in;
  const void* res_in;
  void* res_out;
  void* out;
  const float* weight;
  long long T, H;
  int V;       // 16-byte vectors per row
  int tpr;     // consumer threads per row group (multiple of 32)
  int groups;  // k2_tma_kernel: consumer row groups per CTA (1 or 2; groups * tpr <= 512)
  int stages;  // smem ring depth
  int lookahead;  // k2_tma_kernel: rows of loads in flight ahead of the oldest unarrived one (0 = the ring)
  uint32_t row_bytes;
  float eps;
};

constexpr int kBulkMaxConsumers = 512;

template <class E, int VPT>
__global__ void __launch_bounds__(kBulkMaxConsumers + 32, 1) k2_bulk_kernel(const __grid_constant__ BulkParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.stages;
  unsigned char* ring = smem;  // [S][2][row_bytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * 2 * p.row_bytes);
  uint64_t* empty = full + S;
  Acc* part = reinterpret_cast<Acc*>(empty + S);  // [2][consumer warps]

  const int tpr = p.tpr;
  const int cwarps = tpr >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cwarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const long long nrows = p.T > blockIdx.x ? (p.T - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 0) {
    // ---- producer ----
    if (lane == 0) {
      for (long long i = 0; i < nrows; ++i) {
        const int s = static_cast<int>(i % S);
        const uint32_t ph = static_cast<uint32_t>((i / S) & 1);
        if (i >= S) mbar_wait(&empty[s], ph ^ 1u);
        const long long row = blockIdx.x + i * gridDim.x;
        unsigned char* dst = ring + static_cast<size_t>(s) * 2 * p.row_bytes;
        mbar_arrive_expect_tx(&full[s], 2 * p.row_bytes);
        bulk_g2s(dst, static_cast<const unsigned char*>(p.in) + row * p.row_bytes, p.row_bytes, &full[s]);
        bulk_g2s(dst + p.row_bytes, static_cast<const unsigned char*>(p.res_in) + row * p.row_bytes, p.row_bytes,
                 &full[s]);
      }
    }
    return;
  }

  // ---- consumers ----
  const int lt = threadIdx.x - 32;
  const int cw = warp - 1;
  float w[VPT][N];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = lt + k * tpr;
    if (c < p.V) load_weight<N>(p.weight, static_cast<long long>(c) * N, w[k]);
  }
  for (long long i = 0; i < nrows; ++i) {
    const int s = static_cast<int>(i % S);
    const uint32_t ph = static_cast<uint32_t>((i / S) & 1);
    const long long row = blockIdx.x + i * gridDim.x;
    const long long rowe = row * p.H;
    const unsigned char* src = ring + static_cast<size_t>(s) * 2 * p.row_bytes;
    mbar_wait(&full[s], ph);
    typename VT::Raw rr[VPT];
    Acc ss = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        float x[N], r[N];
        VT::unpack(lds_v4(src + c * 16), x);
        VT::unpack(lds_v4(src + p.row_bytes + c * 16), r);
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = x[j] + r[j];
        rr[k] = VT::pack(r);
        VT::unpack(rr[k], r);
#pragma unroll
        for (int j = 0; j < N; ++j) ss += static_cast<Acc>(r[j]) * static_cast<Acc>(r[j]);
        VT::store(p.res_out, rowe + static_cast<long long>(c) * N, rr[k]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage free for the producer
    ss = warp_sum(ss);
    Acc total;
    if (cwarps == 1) {
      total = ss;
    } else {
      Acc* pp = part + (i & 1) * cwarps;
      if (lane == 0) pp[cw] = ss;
      named_bar_sync(1, tpr);
      total = 0;
      for (int q = 0; q < cwarps; ++q) total += pp[q];
    }
    const float inv = 1.0f / sqrtf(static_cast<float>(total / static_cast<Acc>(p.H)) + p.eps);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) {
        float o[N];
        VT::unpack(rr[k], o);
#pragma unroll
        for (int j = 0; j < N; ++j) o[j] = o[j] * inv * w[k][j];
        VT::store(p.out, rowe + static_cast<long long>(c) * N, VT::pack(o));
      }
    }
  }
}

}  // namespace tw

namespace tw {

// Shared -> global bulk copy (TMA bulk engine), tracked by bulk async-groups.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts_v4(void* p, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(p)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// K2 v2: TMA bulk engine on BOTH sides.  Loads as in k2_bulk_kernel; the
// consumers write r' over the residual slot and the output over the input
// slot of the same stage, and one consumer thread (the "storer") issues two
// shared->global bulk stores per row.  A stage returns to the producer only
// after the bulk engine has finished READING it (bulk_wait_read<1> lags one
// row so the store of row i overlaps the math of row i+1).  The SM's load/
// store units only touch shared memory; HBM traffic is issued by TMA.
// bf16 row math of k2_tma_kernel on packed lanes (sm_100a): r' with add.rn.bf16x2
// (4 instructions per 8 elements instead of unpack + 8 fp32 adds + repack), the
// sum of squares and out = (r' * inv) * w with f32x2 FFMA2/FMUL2.  Same values
// as the scalar path (r' bitwise; ss summed as two interleaved fp32 partials).
// Used with two row groups (the SM-budgeted and short-batch regime, where the
// per-row latency bounds what one SM moves: 72.9 -> 80.5 GB/s per SM at an
// 8-SM budget, H = 8192).  One group keeps the scalar path: with the packed
// path a long batch (T = 16384, H = 8192) measured 178 vs 161 us
// (profiles/k2_packed_ab_r02.txt).
template <int VPT>
__device__ __forceinline__ float k2_bf16_pass1(unsigned char* st, uint32_t row_bytes, int lt, int tpr, int V,
                                               uint4 (&rr)[VPT]) {
  float2 ss = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = lt + k * tpr;
    if (c < V) {
      const uint4 a = lds_v4(st + c * 16);
      const uint4 b = lds_v4(st + row_bytes + c * 16);
      uint4 r;
      r.x = add_bf16x2(a.x, b.x);
      r.y = add_bf16x2(a.y, b.y);
      r.z = add_bf16x2(a.z, b.z);
      r.w = add_bf16x2(a.w, b.w);
      rr[k] = r;
      sts_v4(st + row_bytes + c * 16, r);  // r' over the residual slot
      float2 f = bf16x2_to_f32x2(r.x);
      ss = __ffma2_rn(f, f, ss);
      f = bf16x2_to_f32x2(r.y);
      ss = __ffma2_rn(f, f, ss);
      f = bf16x2_to_f32x2(r.z);
      ss = __ffma2_rn(f, f, ss);
      f = bf16x2_to_f32x2(r.w);
      ss = __ffma2_rn(f, f, ss);
    }
  }
  return ss.x + ss.y;
}

template <int VPT>
__device__ __forceinline__ void k2_bf16_pass2(unsigned char* st, int lt, int tpr, int V, const uint4 (&rr)[VPT],
                                              const float (&w)[VPT][8], float inv) {
  const float2 inv2 = make_float2(inv, inv);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = lt + k * tpr;
    if (c < V) {
      const uint32_t in[4] = {rr[k].x, rr[k].y, rr[k].z, rr[k].w};
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float2 f = __fmul2_rn(bf16x2_to_f32x2(in[q]), inv2);
        f = __fmul2_rn(f, make_float2(w[k][2 * q], w[k][2 * q + 1]));
        o[q] = pack_bf16x2(f.x, f.y);
      }
      sts_v4(st + c * 16, make_uint4(o[0], o[1], o[2], o[3]));  // output over the input slot
    }
  }
}

template <class E, int VPT, int G>
__global__ void __launch_bounds__(kBulkMaxConsumers + 32, 1) k2_tma_kernel(const __grid_constant__ BulkParams p) {
  // G (template: 1 or 2) consumer row groups: group g takes the CTA's rows i = g, g+G, ... (stage
  // i % S), with its own named barrier, partial-sum slots and storer thread,
  // so G rows are normalised concurrently per SM while the ring keeps up to S
  // rows of loads in flight.  G = 2 roughly doubles what one SM moves when the
  // SM count is budgeted (the weave's boundary op); one CTA per SM either way.
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = p.stages;
  unsigned char* ring = smem;  // [S][2][row_bytes]: slot 0 input/output, slot 1 residual/r'
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * 2 * p.row_bytes);
  uint64_t* empty = full + S;
  Acc* part = reinterpret_cast<Acc*>(empty + S);  // [G][2][consumer warps per group]

  const int tpr = p.tpr;
  const int cwarps = tpr >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // released by the storer of the row that used it
    }
    mbar_fence_init();
    k2_tr(0);
  }
  __syncthreads();
  const long long nrows = p.T > blockIdx.x ? (p.T - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 0) {
    if (lane == 0) {
      // Lookahead L < S: row i is requested only once row i - L has ARRIVED,
      // so at most L rows per SM are in flight.  When every SM requests its
      // whole ring at once (short batches: T = 1024 is 7 rows per SM), the
      // memory system interleaves all 148 x S rows and each SM's first row
      // completes near the end of the read phase, leaving the consumers idle
      // until then; a capped lookahead lets the first rows land early and the
      // normalisation overlap the rest of the reads.  The stage of row i - L
      // cannot have been refilled yet (this thread issues in order and L < S),
      // so its full barrier has completed at most once: the parity wait is exact.
      auto issue = [&](long long i, int s) {
        const long long row = blockIdx.x + i * gridDim.x;
        unsigned char* dst = ring + static_cast<size_t>(s) * 2 * p.row_bytes;
        mbar_arrive_expect_tx(&full[s], 2 * p.row_bytes);
        bulk_g2s(dst, static_cast<const unsigned char*>(p.in) + row * p.row_bytes, p.row_bytes, &full[s]);
        bulk_g2s(dst + p.row_bytes, static_cast<const unsigned char*>(p.res_in) + row * p.row_bytes, p.row_bytes,
                 &full[s]);
        if (i < 8) k2_tr(1 + static_cast<int>(i));
      };
      const int L = p.lookahead;
      if (L > 0 && L < S) {
        for (long long i = 0; i < nrows; ++i) {
          const int s = static_cast<int>(i % S);
          if (i >= S) mbar_wait(&empty[s], static_cast<uint32_t>((i / S) & 1) ^ 1u);
          if (i >= L) {
            const long long j = i - L;
            mbar_wait(&full[j % S], static_cast<uint32_t>((j / S) & 1));
          }
          issue(i, s);
        }
      } else {  // the whole ring in flight (kept as its own loop: the refill path is latency-critical)
        for (long long i = 0; i < nrows; ++i) {
          const int s = static_cast<int>(i % S);
          if (i >= S) mbar_wait(&empty[s], static_cast<uint32_t>((i / S) & 1) ^ 1u);
          issue(i, s);
        }
      }
    }
    return;
  }

  const int grp = G == 1 ? 0 : (threadIdx.x - 32) / tpr;
  const int lt = threadIdx.x - 32 - grp * tpr;
  const int cw = lt >> 5;
  const bool storer = lt == 0;
  float w[VPT][N];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = lt + k * tpr;
    if (c < p.V) load_weight<N>(p.weight, static_cast<long long>(c) * N, w[k]);
  }
  if (lt == 0) k2_tr_after(40 + grp, w[0][0]);  // weights in registers
  const float inv_h = 1.0f / static_cast<float>(p.H);
  for (long long i = grp; i < nrows; i += G) {
    const int s = static_cast<int>(i % S);
    const uint32_t ph = static_cast<uint32_t>((i / S) & 1);
    const long long row = blockIdx.x + i * gridDim.x;
    unsigned char* st = ring + static_cast<size_t>(s) * 2 * p.row_bytes;
    mbar_wait(&full[s], ph);
    if (lt == 0 && i < 8) k2_tr(10 + static_cast<int>(i));
    typename VT::Raw rr[VPT];
    Acc ss = 0;
    if constexpr (sizeof(E) == 2 && G == 2) {
      ss = k2_bf16_pass1<VPT>(st, p.row_bytes, lt, tpr, p.V, rr);
    } else {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int c = lt + k * tpr;
        if (c < p.V) {
          float x[N], r[N];
          VT::unpack(lds_v4(st + c * 16), x);
          VT::unpack(lds_v4(st + p.row_bytes + c * 16), r);
#pragma unroll
          for (int j = 0; j < N; ++j) r[j] = x[j] + r[j];
          rr[k] = VT::pack(r);
          VT::unpack(rr[k], r);
#pragma unroll
          for (int j = 0; j < N; ++j) ss += static_cast<Acc>(r[j]) * static_cast<Acc>(r[j]);
          sts_v4(st + p.row_bytes + c * 16, rr[k]);  // r' over the residual slot
        }
      }
    }
    if (lt == 0 && i < 4) k2_tr_after(44 + 4 * static_cast<int>(i), static_cast<float>(ss));
    ss = warp_sum(ss);
    Acc* pp = part + (grp * 2 + ((i / G) & 1)) * cwarps;
    if (lane == 0) pp[cw] = ss;
    constexpr bool kEarlyResStore = sizeof(E) == 2 && G == 2;
    if constexpr (kEarlyResStore) fence_proxy_async_smem();  // r' (pass 1) -> visible to the bulk engine
    named_bar_sync(G == 1 ? 1 : 1 + grp, tpr);
    // r' is final after pass 1: its bulk store starts now and overlaps the
    // statistic and pass 2 (committed with the output's store below)
    if constexpr (kEarlyResStore)
      if (storer)
        bulk_s2g(static_cast<unsigned char*>(p.res_out) + row * p.row_bytes, st + p.row_bytes, p.row_bytes);
    float inv;
    if constexpr (sizeof(E) == 2 && G == 2) {
      // the packed bf16 body (2e-2 tolerance): the warps' partials as 16-byte
      // loads and a tree, and one rsqrt -- the serial chain of dependent
      // shared loads + IEEE div/sqrt/div sits on every row's critical path
      float total = 0.0f;
      if ((cwarps & 3) == 0) {
        for (int q = 0; q < cwarps; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(pp + q);
          total += (v.x + v.y) + (v.z + v.w);
        }
      } else {
        for (int q = 0; q < cwarps; ++q) total += pp[q];
      }
      inv = rsqrtf(total * inv_h + p.eps);
    } else {
      Acc total = 0;
      for (int q = 0; q < cwarps; ++q) total += pp[q];
      inv = 1.0f / sqrtf(static_cast<float>(total / static_cast<Acc>(p.H)) + p.eps);
    }
    if (lt == 0 && i < 4) k2_tr_after(45 + 4 * static_cast<int>(i), inv);
    if constexpr (sizeof(E) == 2 && G == 2) {
      k2_bf16_pass2<VPT>(st, lt, tpr, p.V, rr, w, inv);
    } else {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int c = lt + k * tpr;
        if (c < p.V) {
          float o[N];
          VT::unpack(rr[k], o);
#pragma unroll
          for (int j = 0; j < N; ++j) o[j] = o[j] * inv * w[k][j];
          sts_v4(st + c * 16, VT::pack(o));  // output over the input slot
        }
      }
    }
    if (lt == 0 && i < 4) k2_tr(46 + 4 * static_cast<int>(i));
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk engine
    named_bar_sync(G == 1 ? 1 : 1 + grp, tpr);
    if (lt == 0 && i < 4) k2_tr(47 + 4 * static_cast<int>(i));
    if (storer) {
      bulk_s2g(static_cast<unsigned char*>(p.out) + row * p.row_bytes, st, p.row_bytes);
      if constexpr (!kEarlyResStore)
        bulk_s2g(static_cast<unsigned char*>(p.res_out) + row * p.row_bytes, st + p.row_bytes, p.row_bytes);
      bulk_commit();
      if (i < 8) k2_tr(20 + static_cast<int>(i));
      // this storer's previous row (i - G) has finished reading its stage: free
      // it (a one-row lag, so the store overlaps the next row's math; freeing
      // each stage as soon as it is read stalls the group: -10-20 %,
      // profiles/k2_engines_r01.txt)
      if (i >= G) {
        bulk_wait_read<1>();
        mbar_arrive(&empty[(i - G) % S]);
      }
    }
  }
  if (storer) {
    // The stage must stay valid until the bulk engine has READ it; completion
    // of the global writes is ordered by the kernel boundary (as CUTLASS's TMA
    // store epilogues end on wait_group.read 0).
    bulk_wait_read<0>();
    k2_tr(30 + grp);
    if (nrows > grp) mbar_arrive(&empty[(grp + (nrows - 1 - grp) / G * G) % S]);
  }
}

}  // namespace tw
