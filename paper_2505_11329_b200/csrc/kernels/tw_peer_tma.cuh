// tw_peer_tma.cuh -- K1 over the PEER transport as a bulk-copy pipeline (the
// K2 TMA engine's structure, tw_bulk.cuh) for small worlds (W <= 4).
//
// Per owned token row: the producer thread bulk-loads the W ranks' INPUT rows
// and this rank's residual row into one ring stage ((W+1) rows); 256 consumer
// threads sum the W partial rows in rank-ascending fp32 order from 0.0f (the
// reference's order, proj/src/collectives.cpp:74-78, so residuals stay
// bitwise), add the residual, write r' over the residual slot and the normed
// output over slot 0, and the storer thread bulk-stores r' to the local shard,
// the output to every rank's OUTPUT (and r' to every rank's RESIDUAL with
// G = 2).  The rank barriers are the row engine's (tw_rownorm.cuh).
#pragma once

#include "tw_bulk.cuh"
#include "tw_rownorm.cuh"

namespace tw {

constexpr int kPeerTmaMaxWorld = 4;

template <class E, int VPT, int W>
__global__ void __launch_bounds__(256 + 32, 1) k1_peer_tma_kernel(const __grid_constant__ RowParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  const RankSlot& s = p.slot[blockIdx.y];
  const int S = p.nslots_stages;  // ring depth
  const uint32_t row_bytes = static_cast<uint32_t>(p.H * sizeof(E));
  const size_t stage_bytes = static_cast<size_t>(W + 1) * row_bytes;
  unsigned char* ring = smem;  // [S][W inputs | residual]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * stage_bytes);
  uint64_t* empty = full + S;
  Acc* part = reinterpret_cast<Acc*>(empty + S);  // [2][8 consumer warps]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int tpr = 256;
  constexpr int cwarps = tpr / 32;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  rank_barrier<Xport::Peer>(p, s, 1);  // includes __syncthreads (mbarrier init visible)

  const long long row0 = s.begin, row1 = s.end;
  const long long stride = gridDim.x;
  const long long nrows = row1 - row0 > blockIdx.x ? (row1 - row0 - 1 - blockIdx.x) / stride + 1 : 0;

  if (warp == 0) {
    if (lane == 0) {
      for (long long i = 0; i < nrows; ++i) {
        const int st = static_cast<int>(i % S);
        const uint32_t ph = static_cast<uint32_t>((i / S) & 1);
        if (i >= S) mbar_wait(&empty[st], ph ^ 1u);
        const long long t = row0 + blockIdx.x + i * stride;
        unsigned char* dst = ring + static_cast<size_t>(st) * stage_bytes;
        mbar_arrive_expect_tx(&full[st], (W + 1) * row_bytes);
#pragma unroll
        for (int q = 0; q < W; ++q)
          bulk_g2s(dst + q * row_bytes,
                   static_cast<const unsigned char*>(p.peer_in[q]) + (p.row_offset + t) * row_bytes, row_bytes,
                   &full[st]);
        bulk_g2s(dst + W * row_bytes, static_cast<const unsigned char*>(s.residual) + (t - row0) * row_bytes,
                 row_bytes, &full[st]);
      }
    }
  } else {
    const int lt = threadIdx.x - 32;
    const int cw = lt >> 5;
    const bool storer = lt == 0;
    float w[VPT][N];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) load_weight<N>(s.weight, static_cast<long long>(c) * N, w[k]);
    }
    for (long long i = 0; i < nrows; ++i) {
      const int st = static_cast<int>(i % S);
      const uint32_t ph = static_cast<uint32_t>((i / S) & 1);
      const long long t = row0 + blockIdx.x + i * stride;
      unsigned char* stg = ring + static_cast<size_t>(st) * stage_bytes;
      unsigned char* res = stg + W * row_bytes;
      mbar_wait(&full[st], ph);
      typename VT::Raw rr[VPT];
      Acc ss = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int c = lt + k * tpr;
        if (c < p.V) {
          float x[N], r[N];
#pragma unroll
          for (int j = 0; j < N; ++j) x[j] = 0.0f;
#pragma unroll
          for (int q = 0; q < W; ++q) {  // rank-ascending fp32 sum from 0.0f
            float f[N];
            VT::unpack(lds_v4(stg + q * row_bytes + c * 16), f);
#pragma unroll
            for (int j = 0; j < N; ++j) x[j] += f[j];
          }
          VT::unpack(lds_v4(res + c * 16), r);
#pragma unroll
          for (int j = 0; j < N; ++j) r[j] = x[j] + r[j];
          rr[k] = VT::pack(r);
          VT::unpack(rr[k], r);
#pragma unroll
          for (int j = 0; j < N; ++j) ss += static_cast<Acc>(r[j]) * static_cast<Acc>(r[j]);
          sts_v4(res + c * 16, rr[k]);  // r' over the residual slot
        }
      }
      ss = warp_sum(ss);
      Acc* pp = part + (i & 1) * cwarps;
      if (lane == 0) pp[cw] = ss;
      named_bar_sync(1, tpr);
      Acc total = 0;
      for (int q = 0; q < cwarps; ++q) total += pp[q];
      const float inv = 1.0f / sqrtf(static_cast<float>(total / static_cast<Acc>(p.H)) + p.eps);
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int c = lt + k * tpr;
        if (c < p.V) {
          float o[N];
          VT::unpack(rr[k], o);
#pragma unroll
          for (int j = 0; j < N; ++j) o[j] = o[j] * inv * w[k][j];
          sts_v4(stg + c * 16, VT::pack(o));  // output over input slot 0
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, tpr);
      if (storer) {
        const long long grow = (p.row_offset + t) * row_bytes;
        bulk_s2g(static_cast<unsigned char*>(s.residual) + (t - row0) * row_bytes, res, row_bytes);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          bulk_s2g(static_cast<unsigned char*>(p.peer_out[q]) + grow, stg, row_bytes);
          if (p.flags & kGatherResidual) bulk_s2g(static_cast<unsigned char*>(p.peer_res[q]) + grow, res, row_bytes);
        }
        bulk_commit();
        if (i > 0) {
          bulk_wait_read<1>();
          mbar_arrive(&empty[(i - 1) % S]);
        }
      }
    }
    if (storer) {
      bulk_wait_all();  // every store performed before the exit barrier signals
      asm volatile("fence.proxy.async.global;" ::: "memory");
      fence_acq_rel_sys();
    }
  }
  rank_barrier<Xport::Peer>(p, s, 2);
}

}  // namespace tw
