// tw_weave.cu -- the token-split weave as real CUDA streams (libtw_weave.so).
//
// The reference builds this DAG only to price it in a simulator
// (proj/src/scheduler.cpp:109-183, simulate :185-299).  Here every node is a
// real launch: cuBLAS bf16 GEMMs for the synthetic attention / FFN load on the
// compute stream (library work, not the product) and the fused boundary op
// from libtw.so on a highest-priority stream; every DAG edge is a cudaEvent.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <vector>

#include "tw/tw.h"
#include "tw/tw_split.h"
#include "tw/tw_weave.h"
#include "tw/tw_workload.h"

namespace {

thread_local char g_err[512];

tw_status werr(tw_status st, const std::string& msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg.c_str());
  std::fprintf(stderr, "tw_weave: %s\n", g_err);
  return st;
}

#define CUDA_TRY(expr)                                                             \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) return werr(TW_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CUBLAS_TRY(expr)                                                           \
  do {                                                                             \
    cublasStatus_t s_ = (expr);                                                    \
    if (s_ != CUBLAS_STATUS_SUCCESS) return werr(TW_ERR_CUDA, std::string(#expr) + ": cublas status " + std::to_string(s_)); \
  } while (0)

#define TW_TRY(expr)                                                               \
  do {                                                                             \
    tw_status t_ = (expr);                                                         \
    if (t_ != TW_OK) return werr(t_, std::string(#expr) + ": " + tw_last_error()); \
  } while (0)

struct Ev {
  int op, split, stream;
  cudaEvent_t start, end;
};

}  // namespace

struct tw_weave {
  tw_layer_spec spec;
  int64_t max_tokens = 0;
  int device = 0;
  cublasHandle_t blas = nullptr;
  cudaStream_t compute = nullptr, boundary = nullptr;
  // activations (bf16)
  void *X = nullptr, *P = nullptr, *R = nullptr, *QKV = nullptr, *S = nullptr, *A = nullptr, *F = nullptr,
       *PE = nullptr;
  // weights (bf16) + norm weight (fp32)
  void *Wqkv = nullptr, *Wo = nullptr, *Wup = nullptr, *Wdown = nullptr;
  float* wnorm = nullptr;
  int64_t qkvw = 0, hg = 0, ffn_w = 0, moe_rows = 0;
  std::vector<Ev> pool;
  size_t pool_used = 0;
  std::vector<size_t> last_layer_events;
  bool tracing = true;  // per-op timing events (off while capturing a CUDA graph)
  cudaEvent_t t0 = nullptr;
  std::vector<cudaEvent_t> dag;  // edge events
  size_t dag_used = 0;
  // TP >= 2 (multi-process communicator): P is this rank's symmetric INPUT,
  // the fused op writes the replicated normed hidden into OUTPUT, R holds
  // this rank's residual shard rows of every split (full [T,H] addressing).
  tw_comm_t comm = nullptr;
  int rank = 0, world = 1;
  void* X_local = nullptr;  // TP=1 / unfused-baseline hidden buffer
  void* X_comm = nullptr;   // comm OUTPUT
  // Prior-context attention (serving batches, tw_weave_run_batch): a synthetic
  // KV cache of kv_cap tokens x this GPU's KV heads, its score scratch and the
  // context output.  Grown on demand outside timed regions.
  int64_t kv_context = 0;
  int64_t kv_cap = 0;
  // Communication emulation (tw_weave_emulate_comm): published per-token
  // latency tables of the TP boundary ops; empty = run the real op.
  std::vector<double> emu_tokens, emu_fused_us, emu_ar_us;
  int emu_sms = 16;
  int prio_hi = 0;  // greatest stream priority (the boundary stream's)
  std::map<int64_t, int> tuned_budget;  // tw_weave_throughput's auto boundary budget, per batch size
  void *KV = nullptr, *SC = nullptr, *CO = nullptr;
};

namespace {

constexpr size_t kBf16 = 2;

// Row-major C[M,N] = A[M,K] * B[K,N] (bf16 in, fp32 accumulate), batched.
cublasStatus_t gemm_rm(cublasHandle_t h, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t sA,
                       const void* B, int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, int batch) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return CUBLAS_STATUS_SUCCESS;
  const float alpha = 1.0f, beta = 0.0f;
  return cublasGemmStridedBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(N), static_cast<int>(M),
                                    static_cast<int>(K), &alpha, B, CUDA_R_16BF, static_cast<int>(ldb), sB, A,
                                    CUDA_R_16BF, static_cast<int>(lda), sA, &beta, C, CUDA_R_16BF,
                                    static_cast<int>(ldc), sC, batch, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

cudaEvent_t edge(tw_weave* w) {
  if (w->dag_used == w->dag.size()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    w->dag.push_back(e);
  }
  return w->dag[w->dag_used++];
}

size_t op_begin(tw_weave* w, int op, int split, int stream_id, cudaStream_t s) {
  if (!w->tracing) return 0;  // CUDA-graph capture: no per-op timing events
  if (w->pool_used == w->pool.size()) {
    Ev e{};
    cudaEventCreate(&e.start);
    cudaEventCreate(&e.end);
    w->pool.push_back(e);
  }
  Ev& e = w->pool[w->pool_used];
  e.op = op;
  e.split = split;
  e.stream = stream_id;
  cudaEventRecord(e.start, s);
  return w->pool_used++;
}

void op_end(tw_weave* w, size_t id, cudaStream_t s) {
  if (w->tracing) cudaEventRecord(w->pool[id].end, s);
}

// ---- layer ops -------------------------------------------------------------------

// Attention for query rows [r0, r0+n) with kv_prior earlier context tokens:
// QKV projection, the causal attention core as two batched GEMMs over the
// heads of this GPU with L = kv_prior + n/2 keys (flops = 4*h*d*(n^2/2 +
// n*kv_prior), proj/src/wavemodel.cpp:150-153), and the O projection into
// the partial-sum buffer P (the tensor the boundary op all-reduces).
//
// kv_ctx > 0 adds attention over kv_ctx cached prior-context tokens (decode
// tokens' histories, earlier prefill chunks): per KV head of this GPU one
// [g x d] x [d x kv_ctx] and one [g x kv_ctx] x [kv_ctx x d] GEMM (g = query
// heads per KV head), i.e. 4*h*d*kv_ctx flops and kv_ctx*2*(kv_width/tp)*2
// bytes of K/V streamed from HBM -- the reference's prior-context term
// (wavemodel.cpp:154-162, scheduler.cpp:72-83).
tw_status attention(tw_weave* w, int64_t r0, int64_t n, int64_t kv_prior, int64_t kv_ctx = 0) {
  if (n <= 0) return TW_OK;
  const tw_layer_spec& sp = w->spec;
  const int64_t H = sp.hidden, d = sp.head_dim;
  const int64_t L = std::max<int64_t>(1, kv_prior + n / 2);
  char* X = static_cast<char*>(w->X);
  char* QKV = static_cast<char*>(w->QKV);
  char* A = static_cast<char*>(w->A);
  char* P = static_cast<char*>(w->P);
  CUBLAS_TRY(gemm_rm(w->blas, n, w->qkvw, H, X + r0 * H * kBf16, H, 0, w->Wqkv, w->qkvw, 0,
                     QKV + r0 * w->qkvw * kBf16, w->qkvw, 0, 1));
  // scores[h] = Q_h [n x d] * K_h^T [d x L]   (K_h read as a [d x L] operand)
  CUBLAS_TRY(gemm_rm(w->blas, n, L, d, QKV + r0 * w->qkvw * kBf16, w->qkvw, d, QKV, L, d * L, w->S, L, n * L,
                     static_cast<int>(w->hg)));
  // out[h] = scores[h] [n x L] * V_h [L x d]
  CUBLAS_TRY(gemm_rm(w->blas, n, d, L, w->S, L, n * L, QKV, d, L * d, A + r0 * (w->hg * d) * kBf16, w->hg * d, d,
                     static_cast<int>(w->hg)));
  if (kv_ctx > 0) {
    const int64_t kvh = std::max<int64_t>(1, sp.kv_heads / sp.tp), g = w->hg / kvh;
    char* K = static_cast<char*>(w->KV);
    char* V = K + kv_ctx * kvh * d * kBf16;
    // scores[k] = Q_k [g x d] * K_k [d x kv]; out[k] = scores[k] [g x kv] * V_k [kv x d]
    CUBLAS_TRY(gemm_rm(w->blas, g, kv_ctx, d, QKV + r0 * w->qkvw * kBf16, d, g * d, K, kv_ctx, d * kv_ctx, w->SC,
                       kv_ctx, g * kv_ctx, static_cast<int>(kvh)));
    CUBLAS_TRY(gemm_rm(w->blas, g, d, kv_ctx, w->SC, kv_ctx, g * kv_ctx, V, d, kv_ctx * d, w->CO, d, g * d,
                       static_cast<int>(kvh)));
  }
  CUBLAS_TRY(gemm_rm(w->blas, n, H, w->hg * d, A + r0 * (w->hg * d) * kBf16, w->hg * d, 0, w->Wo, H, 0,
                     P + r0 * H * kBf16, H, 0, 1));
  return TW_OK;
}

// Grow the KV cache / score scratch to hold kv tokens of context.
tw_status ensure_context(tw_weave* w, int64_t kv) {
  if (kv <= w->kv_cap) return TW_OK;
  const tw_layer_spec& sp = w->spec;
  const int64_t d = sp.head_dim, kvh = std::max<int64_t>(1, sp.kv_heads / sp.tp), g = w->hg / kvh;
  const int64_t cap = std::max<int64_t>(kv, 2 * w->kv_cap);
  CUDA_TRY(cudaStreamSynchronize(w->compute));
  CUDA_TRY(cudaStreamSynchronize(w->boundary));
  for (void** p : {&w->KV, &w->SC, &w->CO})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  w->kv_cap = 0;
  const size_t sizes[3] = {size_t(2 * cap * kvh * d * kBf16), size_t(kvh * g * cap * kBf16),
                           size_t(kvh * g * d * kBf16)};
  void** ptrs[3] = {&w->KV, &w->SC, &w->CO};
  for (int i = 0; i < 3; ++i) {
    CUDA_TRY(cudaMalloc(ptrs[i], sizes[i]));
    CUDA_TRY(cudaMemset(*ptrs[i], 0, sizes[i]));
  }
  w->kv_cap = cap;
  return TW_OK;
}

// FFN for rows [r0, r0+n): gate+up [H -> 2I/tp] and down [I/tp -> H] into P.
// MoE: T*top_k/E rows per expert, one batched GEMM pair over the experts
// (uniform routing, proj/src/wavemodel.cpp:169-186).
tw_status ffn(tw_weave* w, int64_t r0, int64_t n) {
  if (n <= 0) return TW_OK;
  const tw_layer_spec& sp = w->spec;
  const int64_t H = sp.hidden, I = sp.intermediate / sp.tp;
  char* X = static_cast<char*>(w->X);
  char* F = static_cast<char*>(w->F);
  char* P = static_cast<char*>(w->P);
  if (sp.experts <= 1) {
    CUBLAS_TRY(gemm_rm(w->blas, n, 2 * I, H, X + r0 * H * kBf16, H, 0, w->Wup, 2 * I, 0, F + r0 * 2 * I * kBf16,
                       2 * I, 0, 1));
    CUBLAS_TRY(gemm_rm(w->blas, n, H, I, F + r0 * 2 * I * kBf16, 2 * I, 0, w->Wdown, H, 0, P + r0 * H * kBf16, H, 0,
                       1));
    return TW_OK;
  }
  const int64_t rows = (n * sp.top_k + sp.experts - 1) / sp.experts;
  CUBLAS_TRY(gemm_rm(w->blas, rows, 2 * I, H, X + r0 * H * kBf16, H, 0, w->Wup, 2 * I, H * 2 * I, F, 2 * I,
                     rows * 2 * I, sp.experts));
  CUBLAS_TRY(gemm_rm(w->blas, rows, H, I, F, 2 * I, rows * 2 * I, w->Wdown, H, I * H, w->PE, H, rows * H,
                     sp.experts));
  return TW_OK;
}

// ---- communication emulation (what-if, NOT the product) -----------------------
// Occupies `sms` SMs for `ns` nanoseconds: 512-thread CTAs holding 160 KB of
// shared memory each, so no GEMM CTA can share their SM while they spin --
// the SM footprint of an NVLink-bound fused op whose duration is taken from a
// published latency table.
constexpr int kEmuSmem = 160 * 1024;
__global__ void __launch_bounds__(512, 1) comm_emulation_kernel(unsigned long long ns) {
  extern __shared__ unsigned char hold[];
  if (threadIdx.x == 0) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      __nanosleep(200);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
    hold[0] = 0;
  }
}

// Piecewise-linear interpolation of a latency table at n tokens (linear
// extrapolation past either end).
double emu_interp(const std::vector<double>& xs, const std::vector<double>& ys, double n) {
  if (xs.size() == 1) return ys[0];
  size_t k = 1;
  while (k + 1 < xs.size() && xs[k] < n) ++k;
  const double t = (n - xs[k - 1]) / (xs[k] - xs[k - 1]);
  return std::max(0.0, ys[k - 1] + t * (ys[k] - ys[k - 1]));
}

tw_status emulate(tw_weave* w, double us, cudaStream_t s) {
  comm_emulation_kernel<<<w->emu_sms, 512, kEmuSmem, s>>>(static_cast<unsigned long long>(us * 1e3));
  CUDA_TRY(cudaGetLastError());
  return TW_OK;
}

// While a CUDA graph is being captured: give the kernel node(s) just captured
// on the boundary stream that stream's priority.  Stream priority is not
// carried into captured kernel nodes, so without this a replayed boundary op
// queues behind the GEMMs' CTAs (the graph is instantiated with
// cudaGraphInstantiateFlagUseNodePriority).
void prioritize_captured(tw_weave* w, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaGraphNode_t* deps = nullptr;
  size_t n = 0;
  if (cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &n) != cudaSuccess ||
      st != cudaStreamCaptureStatusActive)
    return;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(deps[i], &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaLaunchAttributeValue v = {};
    v.priority = w->prio_hi;
    cudaGraphKernelNodeSetAttribute(deps[i], cudaLaunchAttributePriority, &v);
  }
}

// Layer-boundary op on rows [r0, r0+n).
//  * single device: K2 reading the partial sums P, updating the residual R in
//    place and writing the normed hidden X;
//  * TP >= 2: K1 on rows [r0, r0+n) of the communicator's symmetric buffers
//    (token_offset = r0): the split's token_shard_map gives this rank's rows,
//    whose residual lives at R + (r0 + b_rank) * H; the replicated output
//    lands in every rank's OUTPUT (= X).
tw_status fused_op(tw_weave* w, int64_t r0, int64_t n, int budget, cudaStream_t s);

tw_status fused(tw_weave* w, int64_t r0, int64_t n, int budget, cudaStream_t s) {
  const tw_status st = fused_op(w, r0, n, budget, s);
  if (st == TW_OK && s == w->boundary) prioritize_captured(w, s);
  return st;
}

tw_status fused_op(tw_weave* w, int64_t r0, int64_t n, int budget, cudaStream_t s) {
  if (n <= 0) return TW_OK;
  if (!w->emu_tokens.empty()) return emulate(w, emu_interp(w->emu_tokens, w->emu_fused_us, double(n)), s);
  const int64_t H = w->spec.hidden;
  char* P = static_cast<char*>(w->P);
  char* R = static_cast<char*>(w->R);
  char* X = static_cast<char*>(w->X);
  if (w->comm) {
    int64_t ranges[16];
    TW_TRY(tw_token_shard_map(n, w->world, ranges));
    char* shard = R + (r0 + ranges[2 * w->rank]) * H * kBf16;
    TW_TRY(tw_fused_allreduce_rmsnorm(w->comm, n, H, r0, ranges, shard, w->wnorm, 1e-5f, TW_BF16, budget, 0u, s));
    return TW_OK;
  }
  TW_TRY(tw_rmsnorm_residual(P + r0 * H * kBf16, R + r0 * H * kBf16, R + r0 * H * kBf16, X + r0 * H * kBf16,
                             w->wnorm, n, H, 1e-5f, TW_BF16, budget, s));
  return TW_OK;
}

// ---- unfused baseline boundary (NOT the product): residual add, then a
// separate RMSNorm that re-reads r' -- the "AR + RMSNorm" row of the paper
// without the AR (TP = 1), two launches and 5*S bytes instead of 4*S.  Both
// kernels are written to run at HBM speed (16-byte accesses, the RMSNorm row
// held in registers between its two passes), so the weave and the fused op
// are compared against a STRONG separate-kernel baseline (round 1 used a
// scalar 2-byte-load RMSNorm that moved ~2.8 TB/s; bench.py's torch add +
// rms_norm line is the independent cross-check).
__global__ void __launch_bounds__(256) unfused_add_kernel(const uint4* __restrict__ a, uint4* __restrict__ r,
                                                          long long nvec) {
  constexpr int U = 4;  // independent 16-byte loads in flight per thread
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i0 < nvec; i0 += U * stride) {
    uint4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < nvec) {
        x[u] = a[i0 + u * stride];
        y[u] = r[i0 + u * stride];
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * stride >= nvec) continue;
      uint32_t* xs = reinterpret_cast<uint32_t*>(&x[u]);
      uint32_t* ys = reinterpret_cast<uint32_t*>(&y[u]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float lo = __uint_as_float(xs[k] << 16) + __uint_as_float(ys[k] << 16);
        const float hi = __uint_as_float(xs[k] & 0xffff0000u) + __uint_as_float(ys[k] & 0xffff0000u);
        __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
        ys[k] = *reinterpret_cast<uint32_t*>(&v);
      }
      r[i0 + u * stride] = y[u];
    }
  }
}

// One row per 256-thread CTA, VPT 16-byte vectors per thread kept in
// registers: read the row once, block-reduce the sum of squares, write.
template <int VPT>
__global__ void __launch_bounds__(256) unfused_rmsnorm_kernel(const uint4* __restrict__ r, uint4* __restrict__ x,
                                                              const float* __restrict__ w, int V, int H) {
  const uint4* row = r + static_cast<long long>(blockIdx.x) * V;
  uint4* out = x + static_cast<long long>(blockIdx.x) * V;
  uint4 v[VPT];
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * 256;
    if (c < V) {
      v[k] = row[c];
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float lo = __uint_as_float(u[j] << 16), hi = __uint_as_float(u[j] & 0xffff0000u);
        ss += lo * lo + hi * hi;
      }
    }
  }
  __shared__ float part[8];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot += part[i];
  const float inv = rsqrtf(tot / H + 1e-5f);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * 256;
    if (c < V) {
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[k]);
      const float4 w0 = reinterpret_cast<const float4*>(w)[2 * c], w1 = reinterpret_cast<const float4*>(w)[2 * c + 1];
      const float ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      uint4 o;
      uint32_t* os = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(u[j] << 16) * inv * ws[2 * j],
                                                 __uint_as_float(u[j] & 0xffff0000u) * inv * ws[2 * j + 1]);
        os[j] = *reinterpret_cast<uint32_t*>(&b);
      }
      out[c] = o;
    }
  }
}

tw_status unfused(tw_weave* w, int64_t r0, int64_t n, cudaStream_t s) {
  if (n <= 0) return TW_OK;
  const int64_t H = w->spec.hidden;
  char* P = static_cast<char*>(w->P);
  char* R = static_cast<char*>(w->R);
  char* X = static_cast<char*>(w->X);
  if (!w->emu_tokens.empty()) {
    // emulated AllReduce, then the real residual add and RMSNorm over all n rows
    TW_TRY(emulate(w, emu_interp(w->emu_tokens, w->emu_ar_us, double(n)), s));
  } else if (w->comm) {
    // TP >= 2: the one-shot AllReduce (K3) INPUT -> OUTPUT first; the residual
    // is replicated (every rank adds and normalises all rows), as in an
    // unfused engine.
    TW_TRY(tw_allreduce(w->comm, n, H, r0, TW_BF16, 0, s));
    P = static_cast<char*>(w->X_comm);
  }
  const long long nvec = n * H / 8;
  unfused_add_kernel<<<static_cast<int>(std::min<long long>((nvec + 255) / 256, 148 * 8)), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(P + r0 * H * kBf16), reinterpret_cast<uint4*>(R + r0 * H * kBf16), nvec);
  const int V = static_cast<int>(H / 8);  // H % 8 == 0 (LayerSpec hidden sizes)
  const uint4* rr = reinterpret_cast<const uint4*>(R + r0 * H * kBf16);
  uint4* xx = reinterpret_cast<uint4*>(X + r0 * H * kBf16);
  const dim3 grid(static_cast<unsigned>(n));
  if (V <= 256)
    unfused_rmsnorm_kernel<1><<<grid, 256, 0, s>>>(rr, xx, w->wnorm, V, static_cast<int>(H));
  else if (V <= 512)
    unfused_rmsnorm_kernel<2><<<grid, 256, 0, s>>>(rr, xx, w->wnorm, V, static_cast<int>(H));
  else if (V <= 1024)
    unfused_rmsnorm_kernel<4><<<grid, 256, 0, s>>>(rr, xx, w->wnorm, V, static_cast<int>(H));
  else
    unfused_rmsnorm_kernel<8><<<grid, 256, 0, s>>>(rr, xx, w->wnorm, V, static_cast<int>(H));
  CUDA_TRY(cudaGetLastError());
  return TW_OK;
}

}  // namespace

extern "C" {

const char* tw_weave_last_error(void) { return g_err; }

int tw_weave_cublas_version(void) {
  int v = 0;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) == CUBLAS_STATUS_SUCCESS) {
    cublasGetVersion(h, &v);
    cublasDestroy(h);
  }
  return v;
}

tw_status tw_weave_emulate_comm(tw_weave_t w, const int64_t* tokens, const float* fused_us, const float* allreduce_us,
                                int n, int sms) {
  if (!w) return werr(TW_ERR_CONFIG, "weave_emulate_comm: null runner");
  w->emu_tokens.clear();
  w->emu_fused_us.clear();
  w->emu_ar_us.clear();
  if (n <= 0) return TW_OK;  // back to the real boundary op
  if (!tokens || !fused_us || !allreduce_us || sms < 1)
    return werr(TW_ERR_CONFIG, "weave_emulate_comm: null table or sms < 1");
  for (int i = 0; i < n; ++i) {
    if (i > 0 && tokens[i] <= tokens[i - 1])
      return werr(TW_ERR_CONFIG, "weave_emulate_comm: tokens must increase");
    w->emu_tokens.push_back(double(tokens[i]));
    w->emu_fused_us.push_back(fused_us[i]);
    w->emu_ar_us.push_back(allreduce_us[i]);
  }
  w->emu_sms = sms;
  CUDA_TRY(cudaSetDevice(w->device));
  CUDA_TRY(cudaFuncSetAttribute(comm_emulation_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmuSmem));
  return TW_OK;
}

static tw_status weave_create(const tw_layer_spec* spec, int64_t max_tokens, int device, tw_comm_t comm,
                              tw_weave_t* out);

tw_status tw_weave_create(const tw_layer_spec* spec, int64_t max_tokens, int device, tw_weave_t* out) {
  return weave_create(spec, max_tokens, device, nullptr, out);
}

tw_status tw_weave_create_tp(const tw_layer_spec* spec, int64_t max_tokens, tw_comm_t comm, tw_weave_t* out) {
  if (!comm) return werr(TW_ERR_CONFIG, "weave_create_tp: null communicator");
  int rank = -1, device = 0, world = 0;
  TW_TRY(tw_comm_local_rank(comm, &rank, &device));
  TW_TRY(tw_comm_info(comm, &world, nullptr, nullptr));
  if (rank < 0) return werr(TW_ERR_CONFIG, "weave_create_tp: needs a multi-process communicator (one rank here)");
  if (!spec || spec->tp != world) return werr(TW_ERR_CONFIG, "weave_create_tp: spec.tp must equal the world size");
  return weave_create(spec, max_tokens, device, comm, out);
}

static tw_status weave_create(const tw_layer_spec* spec, int64_t max_tokens, int device, tw_comm_t comm,
                              tw_weave_t* out) {
  if (!spec || !out) return werr(TW_ERR_CONFIG, "weave_create: null argument");
  *out = nullptr;
  const tw_layer_spec& sp = *spec;
  if (sp.hidden < 1 || sp.intermediate < 1 || sp.heads < 1 || sp.kv_heads < 1 || sp.head_dim < 1 ||
      sp.heads % sp.kv_heads || sp.experts < 1 || sp.top_k < 1 || sp.top_k > sp.experts || sp.tp < 1 ||
      sp.heads % sp.tp || sp.intermediate % sp.tp || max_tokens < 1)
    return werr(TW_ERR_CONFIG, "weave_create: invalid layer spec (LayerSpec::validate, wavemodel.cpp:23-36)");
  if (sp.hidden % 8)  // the runner's buffers move 16-byte bf16 vectors
    return werr(TW_ERR_CONFIG, "weave_create: hidden must be a multiple of 8");
  CUDA_TRY(cudaSetDevice(device));
  auto* w = new tw_weave();
  w->spec = sp;
  w->max_tokens = max_tokens;
  w->device = device;
  const int64_t H = sp.hidden, T = max_tokens, d = sp.head_dim, I = sp.intermediate / sp.tp;
  w->hg = sp.heads / sp.tp;
  w->qkvw = (H + 2 * sp.kv_heads * d) / sp.tp;
  const int64_t hd = w->hg * d;
  w->moe_rows = (T * sp.top_k + sp.experts - 1) / sp.experts;
  const int64_t frows = sp.experts > 1 ? w->moe_rows * sp.experts : T;
  struct Alloc {
    void** p;
    size_t bytes;
  } allocs[] = {
      {&w->X_local, size_t(T * H * kBf16)},
      {&w->P, size_t(comm ? 16 : T * H * kBf16)},
      {&w->R, size_t(T * H * kBf16)},
      {&w->QKV, size_t(T * std::max(w->qkvw, hd) * kBf16) + size_t(T * d * kBf16)},
      {&w->S, size_t(w->hg * T * T * kBf16)},
      {&w->A, size_t(T * hd * kBf16)},
      {&w->F, size_t(frows * 2 * I * kBf16)},
      {&w->PE, size_t(sp.experts > 1 ? frows * H * kBf16 : 16)},
      {&w->Wqkv, size_t(H * w->qkvw * kBf16)},
      {&w->Wo, size_t(hd * H * kBf16)},
      {&w->Wup, size_t(sp.experts * H * 2 * I * kBf16)},
      {&w->Wdown, size_t(sp.experts * I * H * kBf16)},
      {reinterpret_cast<void**>(&w->wnorm), size_t(H * sizeof(float))},
  };
  for (const Alloc& a : allocs) {
    cudaError_t e = cudaMalloc(a.p, a.bytes);
    if (e == cudaSuccess) e = cudaMemset(*a.p, 0, a.bytes);
    if (e != cudaSuccess) {
      tw_weave_destroy(w);
      return werr(TW_ERR_CUDA, std::string("weave_create: cudaMalloc: ") + cudaGetErrorString(e));
    }
  }
  w->X = w->X_local;
  if (comm) {
    size_t bytes = 0;
    TW_TRY(tw_comm_info(comm, &w->world, nullptr, &bytes));
    TW_TRY(tw_comm_local_rank(comm, &w->rank, nullptr));
    if (bytes < size_t(T * H * kBf16)) {
      tw_weave_destroy(w);
      return werr(TW_ERR_DIMENSION, "weave_create_tp: communicator buffers smaller than max_tokens x hidden");
    }
    cudaFree(w->P);
    TW_TRY(tw_comm_buffer(comm, w->rank, TW_BUF_INPUT, &w->P));      // GEMMs write partial sums here
    TW_TRY(tw_comm_buffer(comm, w->rank, TW_BUF_OUTPUT, &w->X_comm));  // K1 writes the normed hidden here
    w->comm = comm;
    w->X = w->X_comm;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUDA_TRY(cudaStreamCreateWithPriority(&w->compute, cudaStreamNonBlocking, lo));
  CUDA_TRY(cudaStreamCreateWithPriority(&w->boundary, cudaStreamNonBlocking, hi));
  w->prio_hi = hi;
  CUBLAS_TRY(cublasCreate(&w->blas));
  CUBLAS_TRY(cublasSetStream(w->blas, w->compute));
  CUDA_TRY(cudaEventCreate(&w->t0));
  *out = w;
  return TW_OK;
}

tw_status tw_weave_buffer(tw_weave_t w, tw_weave_buf which, void** ptr, size_t* bytes) {
  if (!w || !ptr) return werr(TW_ERR_CONFIG, "weave_buffer: null argument");
  const tw_layer_spec& sp = w->spec;
  const int64_t H = sp.hidden, T = w->max_tokens, I = sp.intermediate / sp.tp;
  size_t n = 0;
  switch (which) {
    case TW_WEAVE_BUF_HIDDEN: *ptr = w->X; n = size_t(T * H * kBf16); break;
    case TW_WEAVE_BUF_RESIDUAL: *ptr = w->R; n = size_t(T * H * kBf16); break;
    case TW_WEAVE_BUF_PARTIAL: *ptr = w->P; n = size_t(T * H * kBf16); break;
    case TW_WEAVE_BUF_W_QKV: *ptr = w->Wqkv; n = size_t(H * w->qkvw * kBf16); break;
    case TW_WEAVE_BUF_W_O: *ptr = w->Wo; n = size_t(w->hg * sp.head_dim * H * kBf16); break;
    case TW_WEAVE_BUF_W_UP: *ptr = w->Wup; n = size_t(sp.experts * H * 2 * I * kBf16); break;
    case TW_WEAVE_BUF_W_DOWN: *ptr = w->Wdown; n = size_t(sp.experts * I * H * kBf16); break;
    case TW_WEAVE_BUF_NORM_WEIGHT: *ptr = w->wnorm; n = size_t(H * sizeof(float)); break;
    default: return werr(TW_ERR_CONFIG, "weave_buffer: unknown buffer");
  }
  if (bytes) *bytes = n;
  return TW_OK;
}

tw_status tw_weave_destroy(tw_weave_t w) {
  if (!w) return TW_OK;
  cudaSetDevice(w->device);
  cudaDeviceSynchronize();
  void* bufs[] = {w->X_local, w->comm ? nullptr : w->P, w->R, w->QKV, w->S, w->A, w->F, w->PE, w->Wqkv, w->Wo,
                  w->Wup, w->Wdown, w->wnorm};  // P / X_comm belong to the communicator in TP mode
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (void* b : {w->KV, w->SC, w->CO})
    if (b) cudaFree(b);
  for (Ev& e : w->pool) {
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.end);
  }
  for (cudaEvent_t e : w->dag) cudaEventDestroy(e);
  if (w->t0) cudaEventDestroy(w->t0);
  if (w->blas) cublasDestroy(w->blas);
  if (w->compute) cudaStreamDestroy(w->compute);
  if (w->boundary) cudaStreamDestroy(w->boundary);
  delete w;
  return TW_OK;
}

}  // extern "C"

namespace {

// One layer's DAG.  carry_a / carry_b: the previous layer's last boundary
// events for the prefix / suffix (cross-layer edges, scheduler.cpp:361-362);
// updated on return.  Records per-op timing events into the pool.
tw_status layer(tw_weave* w, int64_t T, int64_t ta, tw_weave_mode mode, int budget, cudaEvent_t& carry_a,
                cudaEvent_t& carry_b) {
  cudaStream_t cs = w->compute, bs = w->boundary;
  if (mode != TW_MODE_WEAVE) {
    // Sequential chain on one stream: attn -> fused -> ffn -> fused.
    if (carry_a) CUDA_TRY(cudaStreamWaitEvent(cs, carry_a, 0));
    size_t id = op_begin(w, TW_OP_ATTENTION, 2, 0, cs);
    TW_TRY(attention(w, 0, T, 0, w->kv_context));
    op_end(w, id, cs);
    if (mode == TW_MODE_FUSE_ONLY || mode == TW_MODE_UNFUSED) {
      id = op_begin(w, TW_OP_FUSED, 2, 0, cs);
      TW_TRY(mode == TW_MODE_UNFUSED ? unfused(w, 0, T, cs) : fused(w, 0, T, 0, cs));
      op_end(w, id, cs);
    }
    id = op_begin(w, TW_OP_FFN, 2, 0, cs);
    TW_TRY(ffn(w, 0, T));
    op_end(w, id, cs);
    if (mode == TW_MODE_FUSE_ONLY || mode == TW_MODE_UNFUSED) {
      id = op_begin(w, TW_OP_FUSED, 2, 0, cs);
      TW_TRY(mode == TW_MODE_UNFUSED ? unfused(w, 0, T, cs) : fused(w, 0, T, 0, cs));
      op_end(w, id, cs);
    }
    carry_a = edge(w);
    CUDA_TRY(cudaEventRecord(carry_a, cs));
    carry_b = nullptr;
    return TW_OK;
  }
  const int64_t tb = T - ta;
  // prior context divides between the splits in token proportion (scheduler.cpp:124-125)
  const int64_t kv_a = w->kv_context * ta / T, kv_b = w->kv_context - kv_a;
  // compute: attn(a)
  if (carry_a) CUDA_TRY(cudaStreamWaitEvent(cs, carry_a, 0));
  size_t id = op_begin(w, TW_OP_ATTENTION, 0, 0, cs);
  TW_TRY(attention(w, 0, ta, 0, kv_a));
  op_end(w, id, cs);
  cudaEvent_t e_aa = edge(w);
  CUDA_TRY(cudaEventRecord(e_aa, cs));
  // boundary: fused(a) after attn(a)
  CUDA_TRY(cudaStreamWaitEvent(bs, e_aa, 0));
  id = op_begin(w, TW_OP_FUSED, 0, 1, bs);
  TW_TRY(fused(w, 0, ta, budget, bs));
  op_end(w, id, bs);
  cudaEvent_t e_fa1 = edge(w);
  CUDA_TRY(cudaEventRecord(e_fa1, bs));
  // compute: attn(b) -- chunked-attention edge: keys include the prefix
  if (carry_b) CUDA_TRY(cudaStreamWaitEvent(cs, carry_b, 0));
  id = op_begin(w, TW_OP_ATTENTION, 1, 0, cs);
  TW_TRY(attention(w, ta, tb, ta, kv_b));
  op_end(w, id, cs);
  cudaEvent_t e_ab = edge(w);
  CUDA_TRY(cudaEventRecord(e_ab, cs));
  // boundary: fused(b) after attn(b) (and fused(a): same stream)
  CUDA_TRY(cudaStreamWaitEvent(bs, e_ab, 0));
  id = op_begin(w, TW_OP_FUSED, 1, 1, bs);
  TW_TRY(fused(w, ta, tb, budget, bs));
  op_end(w, id, bs);
  cudaEvent_t e_fb1 = edge(w);
  CUDA_TRY(cudaEventRecord(e_fb1, bs));
  // compute: ffn(a) after fused(a)
  CUDA_TRY(cudaStreamWaitEvent(cs, e_fa1, 0));
  id = op_begin(w, TW_OP_FFN, 0, 0, cs);
  TW_TRY(ffn(w, 0, ta));
  op_end(w, id, cs);
  cudaEvent_t e_ffa = edge(w);
  CUDA_TRY(cudaEventRecord(e_ffa, cs));
  // boundary: fused(a) after ffn(a), fused(b)
  CUDA_TRY(cudaStreamWaitEvent(bs, e_ffa, 0));
  id = op_begin(w, TW_OP_FUSED, 0, 1, bs);
  TW_TRY(fused(w, 0, ta, budget, bs));
  op_end(w, id, bs);
  carry_a = edge(w);
  CUDA_TRY(cudaEventRecord(carry_a, bs));
  // compute: ffn(b) after fused(b)
  CUDA_TRY(cudaStreamWaitEvent(cs, e_fb1, 0));
  id = op_begin(w, TW_OP_FFN, 1, 0, cs);
  TW_TRY(ffn(w, ta, tb));
  op_end(w, id, cs);
  cudaEvent_t e_ffb = edge(w);
  CUDA_TRY(cudaEventRecord(e_ffb, cs));
  // boundary: fused(b) after ffn(b), fused(a)
  CUDA_TRY(cudaStreamWaitEvent(bs, e_ffb, 0));
  id = op_begin(w, TW_OP_FUSED, 1, 1, bs);
  TW_TRY(fused(w, ta, tb, budget, bs));
  op_end(w, id, bs);
  carry_b = edge(w);
  CUDA_TRY(cudaEventRecord(carry_b, bs));
  return TW_OK;
}

}  // namespace

namespace {

// `layers` chained layers captured once into a CUDA graph (both streams:
// the boundary stream joins the capture through the DAG's events) and replayed;
// the replay is timed.  Removes the per-launch CPU cost of the ~15 launches
// and event edges per layer.  Valid in TP mode too: the fused op's barrier
// state lives in device memory, so a replayed launch is a fresh launch.
tw_status run_graph(tw_weave* w, int64_t T, int64_t prefix, tw_weave_mode mode, int budget, int gemm_sms,
                    int layers, float* us_per_layer) {
  if (T < 1 || T > w->max_tokens) return werr(TW_ERR_DIMENSION, "weave_run: T out of range");
  if (layers < 1) return werr(TW_ERR_CONFIG, "weave_run: layers must be >= 1");
  if (mode == TW_MODE_WEAVE && (prefix < 1 || prefix >= T))
    return werr(TW_ERR_CONTRACT, "weave_run: TokenWeave requires an Overlap split (0 < prefix < T)");
  CUDA_TRY(cudaSetDevice(w->device));
  CUBLAS_TRY(cublasSetSmCountTarget(w->blas, mode == TW_MODE_WEAVE ? std::max(0, gemm_sms) : 0));
  w->X = (w->comm && mode != TW_MODE_UNFUSED) ? w->X_comm : w->X_local;
  cudaEvent_t ca = nullptr, cb = nullptr;
  w->tracing = false;
  w->dag_used = 0;
  tw_status st = layer(w, T, prefix, mode, budget, ca, cb);  // eager warm-up (cuBLAS setup)
  if (st == TW_OK) {
    cudaError_t e = cudaStreamSynchronize(w->compute);
    if (e == cudaSuccess) e = cudaStreamSynchronize(w->boundary);
    if (e != cudaSuccess) st = werr(TW_ERR_CUDA, std::string("weave graph warm-up: ") + cudaGetErrorString(e));
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  if (st == TW_OK) {
    w->dag_used = 0;
    ca = cb = nullptr;
    cudaError_t e = cudaStreamBeginCapture(w->compute, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) st = werr(TW_ERR_CUDA, std::string("begin capture: ") + cudaGetErrorString(e));
    for (int l = 0; st == TW_OK && l < layers; ++l) st = layer(w, T, prefix, mode, budget, ca, cb);
    if (st == TW_OK) {
      if (cb) cudaStreamWaitEvent(w->compute, cb, 0);
      if (ca) cudaStreamWaitEvent(w->compute, ca, 0);
    }
    e = cudaStreamEndCapture(w->compute, &graph);
    if (st == TW_OK && e != cudaSuccess) st = werr(TW_ERR_CUDA, std::string("end capture: ") + cudaGetErrorString(e));
    if (st == TW_OK) {
      // Per-node priorities: captured kernel nodes carry their stream's
      // priority, but a graph runs every node at the LAUNCH stream's priority
      // (the low-priority compute stream) unless told otherwise -- which
      // would demote the boundary op behind the GEMMs.
      e = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
      if (e != cudaSuccess) st = werr(TW_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
  }
  if (st == TW_OK) {
    cudaEvent_t t1 = nullptr;
    cudaError_t e = cudaGraphLaunch(exec, w->compute);  // warm replay
    if (e == cudaSuccess) e = cudaEventCreate(&t1);
    if (e == cudaSuccess) e = cudaEventRecord(w->t0, w->compute);
    if (e == cudaSuccess) e = cudaGraphLaunch(exec, w->compute);
    if (e == cudaSuccess) e = cudaEventRecord(t1, w->compute);
    if (e == cudaSuccess) e = cudaEventSynchronize(t1);
    float ms = 0;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, w->t0, t1);
    if (t1) cudaEventDestroy(t1);
    if (e != cudaSuccess) st = werr(TW_ERR_CUDA, std::string("graph replay: ") + cudaGetErrorString(e));
    *us_per_layer = 1000.0f * ms / layers;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  w->tracing = true;
  w->last_layer_events.clear();
  cublasSetSmCountTarget(w->blas, 0);
  return st;
}

}  // namespace

extern "C" {

tw_status tw_weave_run(tw_weave_t w, int64_t T, int64_t prefix_tokens, tw_weave_mode mode, int boundary_sm_budget,
                       int gemm_sm_target, int layers, float* us_per_layer) {
  return tw_weave_run_ex(w, T, prefix_tokens, mode, boundary_sm_budget, gemm_sm_target, layers, 0u, us_per_layer);
}

tw_status tw_weave_run_ex(tw_weave_t w, int64_t T, int64_t prefix_tokens, tw_weave_mode mode, int boundary_sm_budget,
                          int gemm_sm_target, int layers, unsigned flags, float* us_per_layer) {
  return tw_weave_run_batch(w, T, prefix_tokens, 0, mode, boundary_sm_budget, gemm_sm_target, layers, flags,
                            us_per_layer);
}

tw_status tw_weave_run_batch(tw_weave_t w, int64_t T, int64_t prefix_tokens, int64_t kv_context, tw_weave_mode mode,
                             int boundary_sm_budget, int gemm_sm_target, int layers, unsigned flags,
                             float* us_per_layer) {
  if (!w || !us_per_layer) return werr(TW_ERR_CONFIG, "weave_run: null argument");
  if (kv_context < 0) return werr(TW_ERR_DIMENSION, "weave_run: negative kv_context");
  CUDA_TRY(cudaSetDevice(w->device));
  if (tw_status st = ensure_context(w, kv_context)) return st;
  w->kv_context = kv_context;
  if (flags & TW_WEAVE_CUDA_GRAPH) return run_graph(w, T, prefix_tokens, mode, boundary_sm_budget, gemm_sm_target,
                                                    layers, us_per_layer);
  if (T < 1 || T > w->max_tokens) return werr(TW_ERR_DIMENSION, "weave_run: T out of range");
  if (layers < 1) return werr(TW_ERR_CONFIG, "weave_run: layers must be >= 1");
  if (mode == TW_MODE_WEAVE && (prefix_tokens < 1 || prefix_tokens >= T))
    return werr(TW_ERR_CONTRACT, "weave_run: TokenWeave requires an Overlap split (0 < prefix < T), "
                                 "scheduler.cpp:116-118");
  CUDA_TRY(cudaSetDevice(w->device));
  CUBLAS_TRY(cublasSetSmCountTarget(w->blas, mode == TW_MODE_WEAVE ? std::max(0, gemm_sm_target) : 0));
  // TP mode: the fused op leaves the normed hidden in the comm OUTPUT; the
  // unfused baseline normalises into a local buffer after the AllReduce.
  w->X = (w->comm && mode != TW_MODE_UNFUSED) ? w->X_comm : w->X_local;
  cudaEvent_t ca = nullptr, cb = nullptr;
  // warm-up layer (cuBLAS heuristics, first-launch costs), not timed
  w->pool_used = 0;
  w->dag_used = 0;
  tw_status st = layer(w, T, prefix_tokens, mode, boundary_sm_budget, ca, cb);
  if (st != TW_OK) return st;
  CUDA_TRY(cudaStreamSynchronize(w->compute));
  CUDA_TRY(cudaStreamSynchronize(w->boundary));
  w->pool_used = 0;
  w->dag_used = 0;
  ca = cb = nullptr;
  CUDA_TRY(cudaEventRecord(w->t0, w->compute));
  CUDA_TRY(cudaStreamWaitEvent(w->boundary, w->t0, 0));
  size_t last_begin = 0;
  for (int l = 0; l < layers; ++l) {
    last_begin = w->pool_used;
    st = layer(w, T, prefix_tokens, mode, boundary_sm_budget, ca, cb);
    if (st != TW_OK) return st;
  }
  // join both streams onto compute, then stop the clock
  if (cb) CUDA_TRY(cudaStreamWaitEvent(w->compute, cb, 0));
  if (ca) CUDA_TRY(cudaStreamWaitEvent(w->compute, ca, 0));
  cudaEvent_t t1 = edge(w);
  cudaEvent_t t1t;
  CUDA_TRY(cudaEventCreate(&t1t));
  (void)t1;
  CUDA_TRY(cudaEventRecord(t1t, w->compute));
  CUDA_TRY(cudaEventSynchronize(t1t));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, w->t0, t1t));
  cudaEventDestroy(t1t);
  *us_per_layer = 1000.0f * ms / layers;
  w->last_layer_events.clear();
  for (size_t i = last_begin; i < w->pool_used; ++i) w->last_layer_events.push_back(i);
  CUBLAS_TRY(cublasSetSmCountTarget(w->blas, 0));
  return TW_OK;
}

tw_status tw_weave_trace(tw_weave_t w, int max_events, int* n_events, int* op, int* split, int* stream,
                         float* start_us, float* end_us) {
  if (!w || !n_events) return werr(TW_ERR_CONFIG, "weave_trace: null argument");
  const int n = static_cast<int>(std::min<size_t>(w->last_layer_events.size(), std::max(0, max_events)));
  *n_events = n;
  for (int i = 0; i < n; ++i) {
    const Ev& e = w->pool[w->last_layer_events[i]];
    float a = 0, b = 0;
    CUDA_TRY(cudaEventElapsedTime(&a, w->t0, e.start));
    CUDA_TRY(cudaEventElapsedTime(&b, w->t0, e.end));
    if (op) op[i] = e.op;
    if (split) split[i] = e.split;
    if (stream) stream[i] = e.stream;
    if (start_us) start_us[i] = 1000.0f * a;
    if (end_us) end_us[i] = 1000.0f * b;
  }
  return TW_OK;
}

// Serving throughput on measured layers: the reference's simulate_throughput
// (workloads.cpp:111-141) with each batch RUN instead of priced.  Batches come
// from form_batches (FCFS chunked prefill, decode first); in TokenWeave mode a
// batch overlaps only if it has prefill tokens and make_split_plan (b200
// geometry, the model's threshold) says Overlap -- otherwise it runs fuse-only,
// as iteration_timeline degrades it (scheduler.cpp:333-341).
tw_status tw_weave_throughput(tw_weave_t w, const tw_request* requests, int64_t n, int64_t chunk_size,
                              tw_weave_mode mode, int64_t threshold_tokens, int num_layers, int layers_measured,
                              int boundary_sm_budget, int gemm_sm_target, unsigned flags,
                              tw_throughput_result* result, double* iteration_latency_s, int64_t max_iterations) {
  if (!w || !result) return werr(TW_ERR_CONFIG, "weave_throughput: null argument");
  if (num_layers < 1 || layers_measured < 1) return werr(TW_ERR_CONFIG, "weave_throughput: layer counts must be >= 1");
  int64_t nb = 0, ns = 0;
  tw_status st = tw_form_batches(requests, n, chunk_size, nullptr, 0, nullptr, 0, &nb, &ns);
  if (st != TW_OK && st != TW_ERR_DIMENSION) return werr(st, std::string("form_batches: ") + tw_workload_last_error());
  std::vector<tw_iteration_batch> batches(static_cast<size_t>(std::max<int64_t>(nb, 1)));
  std::vector<tw_prefill_slice> slices(static_cast<size_t>(std::max<int64_t>(ns, 1)));
  st = tw_form_batches(requests, n, chunk_size, batches.data(), nb, slices.data(), ns, &nb, &ns);
  if (st != TW_OK) return werr(st, std::string("form_batches: ") + tw_workload_last_error());
  *result = tw_throughput_result{};
  for (int64_t k = 0; k < nb; ++k) {
    const tw_iteration_batch& b = batches[static_cast<size_t>(k)];
    if (b.total_tokens > w->max_tokens)
      return werr(TW_ERR_DIMENSION, "weave_throughput: batch of " + std::to_string(b.total_tokens) +
                                        " tokens exceeds the runner's max_tokens");
    tw_weave_mode m = mode;
    int64_t prefix = 0;
    if (mode == TW_MODE_WEAVE) {
      m = TW_MODE_FUSE_ONLY;
      if (b.num_slices > 0) {
        int64_t a = 0, bb = 0, off = 0;
        int pm = 0;
        st = tw_make_split_plan(b.total_tokens, 148, 128, 32, threshold_tokens, &a, &bb, &off, &pm);
        if (st != TW_OK) return werr(st, "weave_throughput: make_split_plan failed");
        if (pm == 2 && bb > 0) {
          m = TW_MODE_WEAVE;
          prefix = a;
        }
      }
    }
    float us = 0.0f;
    if (m == TW_MODE_WEAVE && boundary_sm_budget == TW_WEAVE_AUTO_BUDGET) {
      // the boundary budget that schedules best on THIS box: measured once per
      // batch size over the candidates, then reused (the weave's best budget
      // differs between boxes and with CUDA-graph replay)
      auto it = w->tuned_budget.find(b.total_tokens);
      if (it == w->tuned_budget.end()) {
        float best = 0.0f;
        int best_b = 64;
        for (int cand : {16, 32, 64}) {
          float t = 0.0f;
          st = tw_weave_run_batch(w, b.total_tokens, prefix, b.kv_context, m, cand, gemm_sm_target, layers_measured,
                                  flags, &t);
          if (st != TW_OK) return st;
          if (best == 0.0f || t < best) {
            best = t;
            best_b = cand;
          }
        }
        w->tuned_budget[b.total_tokens] = best_b;
        us = best;
      } else {
        st = tw_weave_run_batch(w, b.total_tokens, prefix, b.kv_context, m, it->second, gemm_sm_target,
                                layers_measured, flags, &us);
      }
    } else {
      st = tw_weave_run_batch(w, b.total_tokens, prefix, b.kv_context, m,
                              boundary_sm_budget == TW_WEAVE_AUTO_BUDGET ? 64 : boundary_sm_budget, gemm_sm_target,
                              layers_measured, flags, &us);
    }
    if (st != TW_OK) return st;
    const double lat = 1e-6 * static_cast<double>(us) * num_layers;
    if (iteration_latency_s && k < max_iterations) iteration_latency_s[k] = lat;
    result->total_seconds += lat;
    result->total_tokens += b.total_tokens;
  }
  result->iterations = nb;
  if (result->total_seconds > 0.0) result->tokens_per_sec = result->total_tokens / result->total_seconds;
  if (nb > 0) result->mean_iteration_latency = result->total_seconds / static_cast<double>(nb);
  return TW_OK;
}

}  // extern "C"
