/*
 * tw.h -- C-ABI of the B200-native TokenWeave hot path (libtw.so).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 * Device pointers are CUDA device addresses on the rank's device; `stream`
 * arguments are cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Every entry point below replaces a reference interface (paths relative to
 * /root/reference); the drop-in C++ API (the include/weavesim headers) is layered
 * on top of these calls and keeps the reference signatures and exceptions.
 *
 * Threading: a communicator is not safe for concurrent mutation (the
 * reference's RankGroup contract); callers serialise calls on a
 * given tw_comm_t.  tw_last_error() is thread-local.
 */
#ifndef TW_TW_H
#define TW_TW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TW_ABI_VERSION 1

#if defined(__GNUC__)
#define TW_API __attribute__((visibility("default")))
#else
#define TW_API
#endif

/* Status codes.  The first four map 1:1 onto the reference exception
 * taxonomy (proj/include/weavesim/errors.hpp:8-23). */
typedef enum tw_status {
  TW_OK = 0,
  TW_ERR_DIMENSION = 1,   /* weavesim::DimensionError  errors.hpp:8   */
  TW_ERR_NUMERIC = 2,     /* weavesim::NumericError    errors.hpp:12  */
  TW_ERR_CONFIG = 3,      /* weavesim::ConfigError     errors.hpp:16  */
  TW_ERR_CONTRACT = 4,    /* weavesim::ContractError   errors.hpp:21  */
  TW_ERR_CUDA = 5,        /* CUDA runtime/driver failure              */
  TW_ERR_TIMEOUT = 6,     /* cross-rank barrier did not complete      */
  TW_ERR_UNSUPPORTED = 7, /* e.g. NVLS requested on a non-NVSwitch box */
  TW_ERR_PARSE = 8        /* weavesim::ParseError      errors.hpp:26 (traces) */
} tw_status;

/* Activation storage type.  Weights are always fp32 (NormParams::weight is
 * std::vector<float>, proj/include/weavesim/numerics.hpp:27-30). */
typedef enum tw_dtype { TW_BF16 = 0, TW_F32 = 1 } tw_dtype;

/* Transport of the fused collective.
 *  NVLS : NVSwitch multicast object (cuMulticastCreate/BindMem); reduce-
 *         scatter with multimem.ld_reduce, all-gather with multimem.st.
 *  PEER : unicast loads/stores on every rank's mapped buffer (NVLink P2P
 *         between GPUs, or plain HBM when several simulated ranks share one
 *         device -- the reference's in-process RankGroup, collectives.hpp:34).
 *  AUTO : NVLS when every rank is on a distinct multicast-capable device,
 *         PEER otherwise.
 *  NVLS_SIM : TEST transport for one GPU.  Simulated ranks sharing a device
 *         run the NVLS kernels themselves (same instantiated control flow:
 *         pipeline, barriers, generations, G = 2) with each multimem
 *         instruction spelled as per-rank loads/stores/reductions.  Never
 *         chosen by AUTO; co-located communicators only. */
typedef enum tw_transport {
  TW_TRANSPORT_AUTO = 0,
  TW_TRANSPORT_NVLS = 1,
  TW_TRANSPORT_PEER = 2,
  TW_TRANSPORT_NVLS_SIM = 3
} tw_transport;

/* Symmetric buffers owned by a communicator (one per rank, same size). */
typedef enum tw_buffer {
  TW_BUF_INPUT = 0,    /* [T,H] partial sums the producer GEMM writes (RankGroup::inputs)      */
  TW_BUF_OUTPUT = 1,   /* [T,H] replicated normed output (fused_allreduce_rmsnorm's return)    */
  TW_BUF_RESIDUAL = 2  /* [T,H] replicated updated residual (TW_GATHER_RESIDUAL only)           */
} tw_buffer;

/* Flags for the fused op. */
#define TW_GATHER_RESIDUAL 0x1u /* G=2: all-gather r' as well as the output  */
/* NVLS kernel: rows of multimem.ld_reduce kept in flight per row group ahead
 * of the row being normalised, d in 1..3 (0 / unset = 2). */
#define TW_NVLS_DEPTH(d) ((((unsigned)(d)) & 0x3u) << 4)

typedef struct tw_comm* tw_comm_t;

/* Library identification. */
TW_API int tw_abi_version(void);
TW_API const char* tw_version(void);
/* Message of the last failing call on this thread ("" if none). */
TW_API const char* tw_last_error(void);
/* Number of CUDA devices visible (0 on a host without a GPU; never fails). */
TW_API int tw_device_count(void);

/* --- TP = 1: fused residual-add + RMSNorm (kernel K2) -----------------------
 * Replaces weavesim::rmsnorm_residual (proj/include/weavesim/numerics.hpp:42-43,
 * proj/src/numerics.cpp:30-64):
 *   residual_out = input + residual;  output = residual_out * rsqrt(mean(residual_out^2)+eps) * weight
 * input/residual/residual_out/output are [T,H] row-major of `dtype`; weight is
 * fp32[H].  residual_out may alias residual (in-place update); no other
 * aliasing.  sm_budget <= 0 means "whole GPU"; > 0 runs on at most that many
 * SMs (one CTA per SM).  Shape errors -> DIMENSION,
 * eps < 0 or NaN -> NUMERIC (numerics.cpp:43-45). */
TW_API tw_status tw_rmsnorm_residual(const void* input, const void* residual, void* residual_out, void* output,
                              const float* weight, int64_t T, int64_t H, float eps, tw_dtype dtype,
                              int sm_budget, void* stream);

/* K2 over HOST buffers (pinned for full speed): chunks of chunk_rows rows
 * (<= 0: ~8 MiB) are pipelined over a ring of streams -- H2D of chunk k+1,
 * the kernel on chunk k and D2H of chunk k-1 overlap.  Work is ordered after
 * `stream`'s prior work and `stream` waits for completion (no host sync). */
TW_API tw_status tw_rmsnorm_residual_host(const void* h_input, const void* h_residual, void* h_residual_out,
                                          void* h_output, const float* h_weight, int64_t T, int64_t H, float eps,
                                          tw_dtype dtype, int64_t chunk_rows, void* stream);

/* Synchronous form for ANY host memory (pageable or pinned), the drop-in's
 * std::vector path: chunks are staged through a pinned ring by a pool of host
 * threads (copy-in of chunk k+1 | H2D | K2 | D2H | copy-out of chunk k-R
 * overlapped), so pageable matrices are not moved by the driver's serial
 * staging.  flags & TW_HOST_CHECK_FINITE: the staging copy also scans the
 * input and residual for NaN/Inf and the call returns TW_ERR_NUMERIC
 * ("TokenMatrix contains NaN/Inf") -- TokenMatrix::validate's check
 * (proj/src/numerics.cpp:25-27) at no extra pass; the outputs are then
 * unspecified.  Returns when the outputs are written. */
#define TW_HOST_CHECK_FINITE 0x1u
TW_API tw_status tw_rmsnorm_residual_host_sync(const void* h_input, const void* h_residual, void* h_residual_out,
                                               void* h_output, const float* h_weight, int64_t T, int64_t H,
                                               float eps, tw_dtype dtype, unsigned flags);

/* tw_rmsnorm_residual_host_sync whose destination rows may still be in
 * preparation: rows_ready[0..n_ready-1] are row counters the caller advances
 * (release stores / __atomic_store_n) from other threads; chunk k's results
 * are copied into h_output / h_residual_out only once every counter has
 * reached the chunk's last row, so the caller's value-initialisation of the
 * destination overlaps the transfers.  Counters must reach T. */
TW_API tw_status tw_rmsnorm_residual_host_sync_gated(const void* h_input, const void* h_residual,
                                                     void* h_residual_out, void* h_output, const float* h_weight,
                                                     int64_t T, int64_t H, float eps, tw_dtype dtype,
                                                     unsigned flags, const int64_t* rows_ready, int n_ready);

/* Device-side finite scan: *nonfinite_count (device int32) += #NaN/Inf in x.
 * Replaces TokenMatrix::validate's isfinite loop (numerics.cpp:25-27). */
TW_API tw_status tw_count_nonfinite(const void* x, int64_t n, tw_dtype dtype, int* nonfinite_count_dev, void* stream);

/* --- Token shard map (host, integer) -----------------------------------------
 * Replaces weavesim::token_shard_map (proj/src/collectives.cpp:26-39) and
 * ShardMap::validate (:14-24).  ranges: 2*world int64 {begin,end}. */
TW_API tw_status tw_token_shard_map(int64_t num_tokens, int world, int64_t* ranges);
TW_API tw_status tw_shard_map_validate(const int64_t* ranges, int world, int64_t total_tokens);

/* Ranks per communicator (the K1/K3 kernels carry every rank's pointers in
 * their launch parameters).  The drop-in C++ API serves wider RankGroups by a
 * chain of K2 launches (weavesim_dropin.cpp); the reference accepts any N >= 2. */
#define TW_MAX_RANKS 8

/* --- Communicator --------------------------------------------------------------
 * One communicator = `world` ranks with symmetric INPUT/OUTPUT/RESIDUAL buffers
 * of `buffer_bytes` each plus signal pads, set up once (multicast objects
 * bound and mapped, peer pointers resolved).  devices[r] is the CUDA device of
 * rank r; devices may repeat (simulated ranks sharing a GPU, PEER transport).
 * Replaces the in-process RankGroup (proj/include/weavesim/collectives.hpp:36-46). */
TW_API tw_status tw_comm_create(int world, const int* devices, size_t buffer_bytes, tw_transport transport,
                         tw_comm_t* out);
TW_API tw_status tw_comm_destroy(tw_comm_t comm);
TW_API tw_status tw_comm_info(tw_comm_t comm, int* world, tw_transport* transport, size_t* buffer_bytes);
/* The rank this process owns and its device (rank = -1: single-process comm). */
TW_API tw_status tw_comm_local_rank(tw_comm_t comm, int* rank, int* device);
TW_API tw_status tw_comm_buffer(tw_comm_t comm, int rank, tw_buffer which, void** device_ptr);
/* Multicast (NVLS) address of a buffer; TW_ERR_UNSUPPORTED on PEER comms. */
TW_API tw_status tw_comm_multicast_buffer(tw_comm_t comm, int rank, tw_buffer which, void** device_ptr);

/* --- Fused AllReduce + residual-add + RMSNorm (kernel K1) ---------------------
 * Replaces weavesim::fused_allreduce_rmsnorm (proj/include/weavesim/collectives.hpp:63-64,
 * proj/src/collectives.cpp:157-182).  For rank r with token shard [b_r,e_r):
 *   x      = sum over ranks of INPUT[t]          (reduce-scatter, t in shard)
 *   r'     = x + residual_shard[t-b_r]            (residual_shard overwritten, :144)
 *   out[t] = r' * rsqrt(mean(r'^2)+eps) * weight  -> OUTPUT[t] on every rank (all-gather)
 *   with TW_GATHER_RESIDUAL also r' -> RESIDUAL[t] on every rank.
 * token_offset: the op covers rows [token_offset, token_offset+T) of the
 *   symmetric buffers (a token split of the weave); shards are relative to it.
 * shard_ranges: 2*world int64 (must satisfy ShardMap::validate, else CONTRACT).
 * residual_shards[r]: device [e_r-b_r, H] of dtype on rank r's device.
 * weights[r]: device fp32[H] on rank r's device.  streams[r]: cudaStream_t.
 * sm_budget: CTAs per rank (1 CTA/SM), the paper's 2-16 SM knob.
 *
 * _group launches every rank this process owns (required when simulated ranks
 * share a device: one launch keeps them co-resident for the in-kernel
 * barrier).  Ranks never run partially: all must be launched. */
TW_API tw_status tw_fused_allreduce_rmsnorm_group(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset,
                                                  const int64_t* shard_ranges,
                                           void* const* residual_shards, const float* const* weights, float eps,
                                           tw_dtype dtype, int sm_budget, unsigned flags, void* const* streams);

/* --- Multi-process communicators (one process per GPU, e.g. torchrun) ---------
 * Every rank calls tw_comm_create_mp with the same world, buffer_bytes and
 * rendezvous_id (a job-unique string, e.g. broadcast by the launcher); rank 0
 * creates the NVLS multicast object and shares it by POSIX fd over an
 * abstract Unix socket.  Collective per-rank calls must be made in the same
 * order with the same shapes on every rank (the signal-pad epochs are
 * device-resident, per CTA index).  transport: NVLS, PEER (cudaIpc-mapped peer
 * buffers, NVLink P2P), or AUTO = NVLS with a collective fallback to PEER. */
TW_API tw_status tw_comm_create_mp(int world, int rank, int device, size_t buffer_bytes, const char* rendezvous_id,
                                   tw_transport transport, tw_comm_t* out);
/* K1 for the rank this process owns (multi-process communicators). */
TW_API tw_status tw_fused_allreduce_rmsnorm(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset,
                                            const int64_t* shard_ranges, void* residual_shard, const float* weight,
                                            float eps, tw_dtype dtype, int sm_budget, unsigned flags, void* stream);
TW_API tw_status tw_allreduce(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, tw_dtype dtype,
                              int sm_budget, void* stream);
/* The rendezvous used by tw_comm_create_mp, exposed for host-side tests: rank
 * 0's `fd` is delivered to every rank as *fd_out (then a barrier). */
TW_API tw_status tw_rendezvous_exchange_fd(const char* rendezvous_id, int world, int rank, int fd, int* fd_out);

/* --- Unfused baselines (NOT the product path) ---------------------------------
 * all_reduce (collectives.cpp:82-88) over the communicator: OUTPUT[t] = sum_r INPUT[t]
 * for every t (one-shot NVLS ld_reduce + multimem.st, or PEER loads). */
TW_API tw_status tw_allreduce_group(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, tw_dtype dtype,
                                    int sm_budget,
                             void* const* streams);

/* --- Device memory helpers (so C/C++ hosts need no CUDA headers) ------------
 * tw_memcpy uses unified addressing (direction inferred); stream NULL = sync. */
TW_API tw_status tw_device_alloc(int device, size_t bytes, void** ptr);
TW_API tw_status tw_device_free(int device, void* ptr);
TW_API tw_status tw_memcpy(void* dst, const void* src, size_t bytes, void* stream);
TW_API tw_status tw_device_synchronize(int device);

/* Host (pageable or pinned) <-> device copies staged through the library's
 * pinned ring by its pool of host threads: 8 MiB chunks, the host copy of one
 * chunk overlapping the DMA of the others (a pageable cudaMemcpy is staged by
 * the driver serially on the calling thread).  Ordered after the legacy
 * default stream's prior work on the device that owns the device pointer;
 * synchronous (return = copy complete).  The drop-in's RankGroup path.
 * h2d: flags & TW_HOST_CHECK_FINITE scans the copied elements (dtype) for
 * NaN/Inf on the way (TokenMatrix::validate's isfinite, numerics.cpp:25-27)
 * and sets *nonfinite (the copy still completes). */
TW_API tw_status tw_memcpy_h2d_staged(void* d_dst, const void* h_src, size_t bytes, tw_dtype dtype, unsigned flags,
                                      int* nonfinite);
TW_API tw_status tw_memcpy_d2h_staged(void* h_dst, const void* d_src, size_t bytes);

/* Per-rank async error flag set by the in-kernel bounded barrier spin.
 * Returns TW_ERR_TIMEOUT (and clears the flag) if any rank timed out. */
TW_API tw_status tw_comm_check(tw_comm_t comm);

#ifdef __cplusplus
}
#endif

#endif /* TW_TW_H */
