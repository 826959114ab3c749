// tw_peer_tma.cuh -- K1 over the PEER transport as a bulk-copy pipeline (the
// K2 TMA engine's structure, tw_bulk.cuh).
//
// Per owned token row the producer thread bulk-loads W + 1 rows -- the W
// ranks' INPUT rows in rank order, then this rank's residual row -- into
// `nchunks` consecutive ring stages (the W + 1 loads split evenly, the larger
// chunks last, so the final stage holds the residual and at least one input
// row).  256 consumer threads sum the W partial rows in rank-ascending fp32
// order from 0.0f in registers across the chunks (the reference's order,
// proj/src/collectives.cpp:74-78, so residuals stay bitwise), add the
// residual, write r' over the residual slot and the normed output over slot 0
// of the final stage, and the storer thread bulk-stores r' to the local
// shard, the output to every rank's OUTPUT (and r' to every rank's RESIDUAL
// with G = 2).  W <= 3 takes one stage per row; W = 4 and W = 8 split a row
// over two stages (2 + 3 and 4 + 5 rows): smaller stages keep the ring 4 and
// 2 deep inside the shared-memory budget (co-located, T = H = 8192: W = 4
// 237 vs 257 us with one stage per row; W = 2 with two stages 184 vs 132 us,
// W = 3 with two 209 vs 181 us, W = 8 with three 384 vs 377 us --
// profiles/k2_engines_r01.txt).  W and the
// chunking are compile-time, so every per-stage sum is unrolled and its
// shared-memory loads issue together.  The rank barriers are the row engine's
// (tw_rownorm.cuh).
#pragma once

#include "tw_bulk.cuh"
#include "tw_rownorm.cuh"

namespace tw {

constexpr int kPeerTmaMaxWorld = kMaxRanks;
__host__ __device__ constexpr int peer_tma_chunks(int W) { return W <= 3 ? 1 : 2; }
__host__ __device__ constexpr int peer_tma_stage_rows(int W) {
  return (W + 1 + peer_tma_chunks(W) - 1) / peer_tma_chunks(W);
}

// G consumer row groups (G = 2 only with one stage per token row, W <= 3):
// group g takes the CTA's rows i = g, g + G, ...; a group frees its stage as
// soon as its stores have read it when the ring has no spare stages for a
// one-row lag.
template <class E, int VPT, int W, int G = 1>
__global__ void __launch_bounds__(G * 256 + 32, 1) k1_peer_tma_kernel(const __grid_constant__ RowParams p) {
  constexpr int N = 16 / sizeof(E);
  using VT = Vec<E, N>;
  using Acc = typename std::conditional<sizeof(E) == 4, double, float>::type;
  constexpr int tpr = 256;
  constexpr int cwarps = tpr / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const RankSlot& s = p.slot[blockIdx.y];
  const int S = p.nslots_stages;  // ring depth (stages)
  constexpr int n = peer_tma_chunks(W);  // stages per row
  constexpr int tot = W + 1;             // row loads per token: W inputs + the residual
  constexpr int base = tot / n, extra = tot % n;
  constexpr int R = peer_tma_stage_rows(W);  // rows per stage (the last chunk is the largest)
  const uint32_t row_bytes = static_cast<uint32_t>(p.H * sizeof(E));
  const size_t stage_bytes = static_cast<size_t>(R) * row_bytes;
  // With more stages than chunks the final stage of a row is released one row
  // late (after the next row's stores are issued); otherwise that would block
  // the producer's next row, so the storer waits for its own reads instead.
  // A parity wait names a phase only if the waiter consumed the stage's
  // previous phase: row i - S must be the group's own row, so S % G == 0
  // (the launcher rounds S down).
  static_assert(G == 1 || peer_tma_chunks(W) == 1, "two row groups need one stage per token row");
  const bool lazy = G == 1 ? S > n : S >= 2 * G + 1;
  unsigned char* ring = smem;  // [S][R rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(S) * stage_bytes);
  uint64_t* empty = full + S;
  Acc* part = reinterpret_cast<Acc*>(empty + S);  // [G][2][8 consumer warps]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], cwarps);
    }
    mbar_fence_init();
  }
  rank_barrier<Xport::Peer>(p, s, 1);  // includes __syncthreads (mbarrier init visible)

  const long long row0 = s.begin, row1 = s.end;
  const long long stride = gridDim.x;
  const long long nrows = row1 - row0 > blockIdx.x ? (row1 - row0 - 1 - blockIdx.x) / stride + 1 : 0;

  if (warp == 0) {
    if (lane == 0) {
      // The entry barrier acquired the peers' INPUT writes through the generic
      // proxy; the bulk loads below read them through the async proxy.
      asm volatile("fence.proxy.async.global;" ::: "memory");
      long long g = 0;  // stage sequence number
      for (long long i = 0; i < nrows; ++i) {
        const long long t = row0 + blockIdx.x + i * stride;
        int item = 0;
#pragma unroll
        for (int c = 0; c < n; ++c, ++g) {
          const int cnt = base + (c >= n - extra ? 1 : 0);
          const int st = static_cast<int>(g % S);
          if (g >= S) mbar_wait(&empty[st], static_cast<uint32_t>(((g / S) & 1) ^ 1));
          unsigned char* dst = ring + static_cast<size_t>(st) * stage_bytes;
          mbar_arrive_expect_tx(&full[st], cnt * row_bytes);
#pragma unroll
          for (int k = 0; k < cnt; ++k, ++item) {
            const unsigned char* src =
                item < W ? static_cast<const unsigned char*>(p.peer_in[item]) + (p.row_offset + t) * row_bytes
                         : static_cast<const unsigned char*>(s.residual) + (t - row0) * row_bytes;
            bulk_g2s(dst + k * row_bytes, src, row_bytes, &full[st]);
          }
        }
      }
    }
  } else {
    const int grp = G == 1 ? 0 : (threadIdx.x - 32) / tpr;
    const int lt = threadIdx.x - 32 - grp * tpr;
    const int cw = lt >> 5;
    const bool storer = lt == 0;
    part += grp * 2 * cwarps;
    float w[VPT][N];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = lt + k * tpr;
      if (c < p.V) load_weight<N>(s.weight, static_cast<long long>(c) * N, w[k]);
    }
    int prev_last = -1;  // final stage of this group's previous row (lazy release)
    for (long long i = grp; i < nrows; i += G) {
      long long g = i * n;  // stage sequence number of the row's first chunk
      const long long t = row0 + blockIdx.x + i * stride;
      float x[VPT][N];
#pragma unroll
      for (int k = 0; k < VPT; ++k)
#pragma unroll
        for (int j = 0; j < N; ++j) x[k][j] = 0.0f;
      // Every chunk but the last holds input rows only: sum, release.
#pragma unroll
      for (int c = 0; c < n - 1; ++c, ++g) {
        const int cnt = base + (c >= n - extra ? 1 : 0);
        const int st = static_cast<int>(g % S);
        mbar_wait(&full[st], static_cast<uint32_t>((g / S) & 1));
        const unsigned char* stg = ring + static_cast<size_t>(st) * stage_bytes;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          const int cc = lt + k * tpr;
          if (cc < p.V) {
#pragma unroll
            for (int q = 0; q < cnt; ++q) {  // rank-ascending fp32 sum from 0.0f
              float f[N];
              VT::unpack(lds_v4(stg + q * row_bytes + cc * 16), f);
#pragma unroll
              for (int j = 0; j < N; ++j) x[k][j] += f[j];
            }
          }
        }
      }
      // The last chunk: the remaining inputs, then the residual row.
      constexpr int cnt = base + (extra ? 1 : 0);
      const int st = static_cast<int>(g % S);
      mbar_wait(&full[st], static_cast<uint32_t>((g / S) & 1));
      ++g;
      unsigned char* stg = ring + static_cast<size_t>(st) * stage_bytes;
      unsigned char* res = stg + (cnt - 1) * row_bytes;
      typename VT::Raw rr[VPT];
      Acc ss = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int cc = lt + k * tpr;
        if (cc < p.V) {
#pragma unroll
          for (int q = 0; q < cnt - 1; ++q) {
            float f[N];
            VT::unpack(lds_v4(stg + q * row_bytes + cc * 16), f);
#pragma unroll
            for (int j = 0; j < N; ++j) x[k][j] += f[j];
          }
          float r[N];
          VT::unpack(lds_v4(res + cc * 16), r);
#pragma unroll
          for (int j = 0; j < N; ++j) r[j] = x[k][j] + r[j];
          rr[k] = VT::pack(r);
          VT::unpack(rr[k], r);
#pragma unroll
          for (int j = 0; j < N; ++j) ss += static_cast<Acc>(r[j]) * static_cast<Acc>(r[j]);
          sts_v4(res + cc * 16, rr[k]);  // r' over the residual slot
        }
      }
      ss = warp_sum(ss);
      Acc* pp = part + (i & 1) * cwarps;
      if (lane == 0) pp[cw] = ss;
      fence_proxy_async_smem();  // r' (written above) -> visible to the bulk engine
      named_bar_sync(1 + grp, tpr);
      const long long grow = (p.row_offset + t) * row_bytes;
      if (storer) {
        // Every consumer is past the input-only stages of this row: free them.
#pragma unroll
        for (int c = 0; c < n - 1; ++c) mbar_arrive_n(&empty[static_cast<int>((g - n + c) % S)], cwarps);
        // r' is final: its stores (the local shard, and every rank's RESIDUAL
        // with G = 2) start now and overlap the statistic and the output pass;
        // they are committed with the output's stores below.
        bulk_s2g(static_cast<unsigned char*>(s.residual) + (t - row0) * row_bytes, res, row_bytes);
        if (p.flags & kGatherResidual) {
#pragma unroll
          for (int q = 0; q < W; ++q) bulk_s2g(static_cast<unsigned char*>(p.peer_res[q]) + grow, res, row_bytes);
        }
      }
      const float inv = inv_rms<Acc>(sum_partials<Acc>(pp, cwarps), p.H, p.eps);
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int cc = lt + k * tpr;
        if (cc < p.V) {
          float o[N];
          VT::unpack(rr[k], o);
#pragma unroll
          for (int j = 0; j < N; ++j) o[j] = o[j] * inv * w[k][j];
          sts_v4(stg + cc * 16, VT::pack(o));  // output over input slot 0
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + grp, tpr);
      if (storer) {
#pragma unroll
        for (int q = 0; q < W; ++q) bulk_s2g(static_cast<unsigned char*>(p.peer_out[q]) + grow, stg, row_bytes);
        bulk_commit();
        if (lazy) {
          if (prev_last >= 0) {
            bulk_wait_read<1>();
            mbar_arrive_n(&empty[prev_last], cwarps);
          }
          prev_last = st;
        } else {
          bulk_wait_read<0>();
          mbar_arrive_n(&empty[st], cwarps);
        }
      }
    }
    if (storer) {
      // Every bulk store performed, then ordered (async -> generic proxy)
      // before this thread's later operations.  No scope fence here: the
      // exit barrier's bar.sync puts these writes before thread 0's
      // fence.acq_rel + red (release pattern, cumulative over the CTA), so
      // one fence per CTA exit publishes them (a second fence here cost a
      // system-scope fence per CTA on the critical path).
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
  rank_barrier<Xport::Peer>(p, s, 2);
}

}  // namespace tw
