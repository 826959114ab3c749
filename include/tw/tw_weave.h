/*
 * tw_weave.h -- C-ABI of the token-split "weave" layer runner (libtw_weave.so).
 *
 * Executes one transformer layer's two-stream DAG on real CUDA streams:
 * synthetic attention / FFN GEMMs (cuBLAS -- load, not product) on a compute
 * stream and the fused layer-boundary op (libtw.so) on a high-priority
 * boundary stream, with a cudaEvent for every DAG edge.  The DAG shapes are
 * the reference's (proj/src/scheduler.cpp:109-183):
 *   TW_MODE_WEAVE      : 8 events, attn(a) -> fused(a) || attn(b) -> fused(b)
 *                        || ffn(a) -> fused(a) || ffn(b) -> fused(b)  (:119-147)
 *   TW_MODE_FUSE_ONLY  : attn -> fused -> ffn -> fused                 (:171-178)
 *   TW_MODE_NO_COMM    : attn -> ffn (boundary op skipped; lower bound) (:165-169)
 * Cross-layer edges fused(a)_L -> attn(a)_{L+1}, fused(b)_L -> attn(b)_{L+1}
 * (:361-362) chain `layers` layers back to back.
 *
 * GEMM shapes are one GPU's share of the layer at tensor-parallel degree
 * `tp` (proj/src/wavemodel.cpp:146-157,173).  The boundary op of this
 * single-device runner is K2 (tw_rmsnorm_residual) over the split's rows --
 * the TP=1 form of the fused op; with tp > 1 it stands in for K1, whose
 * NVLink traffic a single GPU cannot exercise.
 */
#ifndef TW_TW_WEAVE_H
#define TW_TW_WEAVE_H

#include "tw/tw.h"
#include "tw/tw_workload.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tw_layer_spec {
  int64_t hidden;        /* H   */
  int64_t intermediate;  /* I   */
  int32_t heads;         /* attention heads */
  int32_t kv_heads;
  int32_t head_dim;
  int32_t experts;       /* 1 = dense */
  int32_t top_k;
  int32_t tp;            /* GEMM shapes are per GPU at this TP degree */
} tw_layer_spec;

typedef enum tw_weave_mode {
  TW_MODE_FUSE_ONLY = 0,
  TW_MODE_WEAVE = 1,
  TW_MODE_NO_COMM = 2,
  TW_MODE_UNFUSED = 3 /* baseline: attn -> add -> RMSNorm -> ffn -> add -> RMSNorm, one stream
                         (the reference's Multimem chain, scheduler.cpp:153-164, at TP = 1) */
} tw_weave_mode;

/* Ops recorded by tw_weave_trace (the reference's OpKind, scheduler.hpp:12). */
typedef enum tw_weave_op { TW_OP_ATTENTION = 0, TW_OP_FFN = 1, TW_OP_FUSED = 2 } tw_weave_op;

typedef struct tw_weave* tw_weave_t;

/* Message of the last failing call of this header on this thread ("" if none). */
TW_API const char* tw_weave_last_error(void);
/* Version of the cuBLAS the runner's GEMMs actually bind (e.g. 120901 = 12.9.1;
 * 0 without a device).  The process may hold another libcublas.so.12 (torch's)
 * loaded first; DESIGN.md §5. */
TW_API int tw_weave_cublas_version(void);

TW_API tw_status tw_weave_create(const tw_layer_spec* spec, int64_t max_tokens, int device, tw_weave_t* out);
/* TP >= 2 with one process per GPU: `comm` is a multi-process communicator
 * (tw_comm_create_mp, buffers >= max_tokens*hidden*2 B) and spec->tp its world
 * size.  The GEMMs write their partial sums into this rank's INPUT buffer and
 * the boundary op is K1 (tw_fused_allreduce_rmsnorm) on the split's rows;
 * TW_MODE_UNFUSED runs the K3 AllReduce + separate add/RMSNorm instead.
 * Every rank must issue the same tw_weave_run calls. */
TW_API tw_status tw_weave_create_tp(const tw_layer_spec* spec, int64_t max_tokens, tw_comm_t comm,
                                    tw_weave_t* out);
TW_API tw_status tw_weave_destroy(tw_weave_t w);

/* Runs `layers` chained layers of T tokens (prefix_tokens used by WEAVE) and
 * returns the device time per layer in microseconds (CUDA events; warm-up
 * layer excluded).  boundary_sm_budget bounds the fused op's CTAs; when
 * gemm_sm_target > 0 cuBLAS is asked to use that many SMs (the SM partition
 * between compute and boundary work, scheduler.cpp:216-217). */
TW_API tw_status tw_weave_run(tw_weave_t w, int64_t T, int64_t prefix_tokens, tw_weave_mode mode,
                              int boundary_sm_budget, int gemm_sm_target, int layers, float* us_per_layer);

/* tw_weave_run with flags: TW_WEAVE_CUDA_GRAPH captures the `layers` chained
 * layers (both streams, every DAG edge) into one CUDA graph, replays it and
 * times the replay -- no per-launch host cost.  No per-op trace is recorded. */
#define TW_WEAVE_CUDA_GRAPH 0x1u
TW_API tw_status tw_weave_run_ex(tw_weave_t w, int64_t T, int64_t prefix_tokens, tw_weave_mode mode,
                                 int boundary_sm_budget, int gemm_sm_target, int layers, unsigned flags,
                                 float* us_per_layer);

/* tw_weave_run_ex for one serving batch: kv_context prior-context tokens
 * (IterationBatch::kv_context, workloads.hpp:36) are attended from a synthetic
 * KV cache -- 4*h*d*kv_context flops and kv_context*2*(kv_width/tp)*2 bytes,
 * the reference's prior-context term (wavemodel.cpp:154-162); in WEAVE mode
 * they divide between the splits in token proportion (scheduler.cpp:124-125). */
TW_API tw_status tw_weave_run_batch(tw_weave_t w, int64_t T, int64_t prefix_tokens, int64_t kv_context,
                                    tw_weave_mode mode, int boundary_sm_budget, int gemm_sm_target, int layers,
                                    unsigned flags, float* us_per_layer);

/* weavesim::ThroughputResult (workloads.hpp:41-48) without the latency vector. */
typedef struct tw_throughput_result {
  double tokens_per_sec;
  int64_t iterations;
  int64_t total_tokens;
  double total_seconds;
  double mean_iteration_latency;
} tw_throughput_result;

/* Measured serving throughput: the reference's simulate_throughput
 * (proj/src/workloads.cpp:111-141) with every batch of form_batches(requests,
 * chunk_size) RUN through tw_weave_run_batch (layers_measured chained layers
 * after a warm-up layer) and its iteration latency = measured per-layer time x
 * num_layers.  In WEAVE mode decode-only batches and batches make_split_plan
 * (b200 geometry, threshold_tokens) does not split run FUSE_ONLY
 * (scheduler.cpp:333-341).  iteration_latency_s (optional) receives up to
 * max_iterations per-batch latencies in seconds.  boundary_sm_budget =
 * TW_WEAVE_AUTO_BUDGET: for each weaved batch size the fused op's SM budget is
 * measured once over {16, 32, 64} and the fastest reused. */
#define TW_WEAVE_AUTO_BUDGET (-1)
TW_API tw_status tw_weave_throughput(tw_weave_t w, const tw_request* requests, int64_t n, int64_t chunk_size,
                                     tw_weave_mode mode, int64_t threshold_tokens, int num_layers,
                                     int layers_measured, int boundary_sm_budget, int gemm_sm_target,
                                     unsigned flags, tw_throughput_result* result, double* iteration_latency_s,
                                     int64_t max_iterations);

/* What-if (NOT the product): replace the boundary op by an emulation that
 * holds `sms` SMs (512-thread CTAs with 160 KB of shared memory, so no GEMM CTA
 * can share them) for a duration interpolated from a latency table: fused_us
 * for the fused op (FUSE_ONLY / WEAVE), allreduce_us for the AllReduce of the
 * unfused baseline (followed by the real add + RMSNorm kernels).  It lets one
 * GPU measure how the weave schedules a TP = N NVLink-bound op against real
 * cuBLAS GEMMs, with the op's duration taken from a published multi-GPU table.
 * n = 0 restores the real op.  tokens strictly increasing. */
TW_API tw_status tw_weave_emulate_comm(tw_weave_t w, const int64_t* tokens, const float* fused_us,
                                       const float* allreduce_us, int n, int sms);

/* Per-event timestamps (us from the run's start) of the LAST layer of the
 * last tw_weave_run: op (tw_weave_op), split (0 prefix, 1 suffix, 2 whole),
 * stream (0 compute, 1 boundary).  Arrays hold max_events entries. */
TW_API tw_status tw_weave_trace(tw_weave_t w, int max_events, int* n_events, int* op, int* split, int* stream,
                                float* start_us, float* end_us);

/* The runner's device buffers (bf16 unless noted), for tests that seed the
 * layer's weights and read its activations back: the layer's state after a
 * run is what the schedule computed, so two schedules of the same layers can
 * be compared value for value.  HIDDEN is the buffer the current mode's
 * boundary op writes ([max_tokens, H]; in TP mode the comm OUTPUT).
 * *bytes receives the buffer's size. */
typedef enum tw_weave_buf {
  TW_WEAVE_BUF_HIDDEN = 0,     /* X  [max_tokens, H]                      */
  TW_WEAVE_BUF_RESIDUAL = 1,   /* R  [max_tokens, H]                      */
  TW_WEAVE_BUF_PARTIAL = 2,    /* P  [max_tokens, H] (GEMM partial sums)  */
  TW_WEAVE_BUF_W_QKV = 3,      /* [H, qkv_width/tp]                       */
  TW_WEAVE_BUF_W_O = 4,        /* [heads/tp * head_dim, H]                */
  TW_WEAVE_BUF_W_UP = 5,       /* [experts][H, 2*I/tp]                    */
  TW_WEAVE_BUF_W_DOWN = 6,     /* [experts][I/tp, H]                      */
  TW_WEAVE_BUF_NORM_WEIGHT = 7 /* fp32 [H]                                */
} tw_weave_buf;
TW_API tw_status tw_weave_buffer(tw_weave_t w, tw_weave_buf which, void** ptr, size_t* bytes);

#ifdef __cplusplus
}
#endif

#endif
