// tw_launch.h -- host-side launch interface of the row engine (internal).
#pragma once

#include <cuda_runtime.h>

#include "tw_bulk.cuh"
#include "tw_flat.cuh"
#include "tw_nvls.cuh"
#include "tw_peer_tma.cuh"
#include "tw_rownorm.cuh"

namespace tw {

struct RowPlan {
  int N;       // elements per vector (8 bf16 / 4 f32 / 1 scalar)
  int V;       // vectors per row
  int vpt;     // vectors per thread
  int tpr;     // threads per row group
  int groups;  // row groups per CTA
  bool pipeline;  // local engine: software-pipelined row loop (NVLS always pipelines)
};

// Chooses vectors-per-thread and threads-per-row for a row of H elements
// loaded N at a time.  tpr_pref bounds the row-group width (fewer threads per
// row = more rows in flight per CTA).  Returns false if H is unsupported.
// Per (function, device) launch facts, computed once (tw_launch.cu).
int cached_occupancy(const void* fn, int threads, size_t smem);
cudaError_t ensure_dynamic_smem(const void* fn, size_t bytes);

bool plan_rows(long long H, int elems_per_vec, int tpr_pref, RowPlan* plan);

cudaError_t launch_rownorm(const RowParams& params, const RowPlan& plan, bool bf16, Xport x, dim3 grid,
                           cudaStream_t stream);
cudaError_t launch_allreduce(const RowParams& params, const RowPlan& plan, bool bf16, Xport x, dim3 grid,
                             cudaStream_t stream);
int rownorm_blocks_per_sm(const RowPlan& plan, bool bf16, Xport x);
// K1 / K3 over NVLS (tw_nvls.cuh).  sim: the MmSim policy on co-located ranks
// (TW_TRANSPORT_NVLS_SIM); depth: rows of ld_reduce in flight (1..3).
int nvls_depth_from_flags(unsigned flags);
bool nvls_supported(const RowPlan& plan);
cudaError_t launch_k1_nvls(const RowParams& params, const RowPlan& plan, bool bf16, bool sim, int depth, dim3 grid,
                           cudaStream_t stream);
int k1_nvls_blocks_per_sm(const RowPlan& plan, bool bf16, bool sim, int depth);
cudaError_t launch_k3_nvls(const RowParams& params, const RowPlan& plan, bool bf16, bool sim, dim3 grid,
                           cudaStream_t stream);
// K1 over PEER as a bulk-copy pipeline (tw_peer_tma.cuh), 2 <= world <= 8,
// vectorised rows.  Returns cudaErrorNotSupported when the shape does not fit;
// k1_peer_tma_blocks_per_sm returns 0 then (the caller uses the row engine).
cudaError_t launch_k1_peer_tma(RowParams params, int world, int V, bool bf16, dim3 grid, cudaStream_t stream);
int k1_peer_tma_blocks_per_sm(int world, int V, long long H, bool bf16);
size_t bulk_smem_bytes(int stages, uint32_t row_bytes, int tpr, int groups);
cudaError_t launch_k2_bulk(const BulkParams& params, int vpt, bool bf16, int grid, cudaStream_t stream,
                           bool tma_store);
// K2 flat engine (tw_flat.cuh); V <= 2048 vectors per row.
cudaError_t launch_k2_flat(const FlatParams& params, bool bf16, int sms, bool one_cta_per_sm, cudaStream_t stream);
cudaError_t launch_count_nonfinite(const void* x, long long n, bool bf16, int* count, cudaStream_t stream);

}  // namespace tw
