/*
 * tw_oracle.h -- CPU restatement of the reference (weavesim) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker.  The product (libtw.so) never links or calls it.
 *
 * Every function restates a reference routine with the same arithmetic
 * order so the restatement is bit-identical to the reference; the citation
 * next to each declaration is the reference file:line it follows
 * (paths relative to /root/reference).  Parity of this restatement is pinned
 * against oracle/_ref (the reference sources compiled unmodified) and the
 * committed golden fixtures in tests/golden/.
 *
 * Status codes match tw.h: 0 ok, 1 dimension, 2 numeric, 3 config, 4 contract.
 */
#ifndef TW_ORACLE_H
#define TW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_DIMENSION = 1,
  ORC_NUMERIC = 2,
  ORC_CONFIG = 3,
  ORC_CONTRACT = 4
};

/* token_shard_map  proj/src/collectives.cpp:26-39.  ranges: 2*world int64. */
int orc_token_shard_map(int64_t num_tokens, int world, int64_t* ranges);

/* ShardMap::validate  proj/src/collectives.cpp:14-24. */
int orc_shard_map_validate(const int64_t* ranges, int world, int64_t total);

/* TokenMatrix::validate finite scan  proj/src/numerics.cpp:18-28. */
int orc_all_finite(const float* v, int64_t n);

/* rmsnorm_residual  proj/src/numerics.cpp:30-64 (fp32, double sum of squares). */
int orc_rmsnorm_residual(const float* input, const float* residual, const float* weight,
                         int64_t T, int64_t H, float eps, float* output, float* residual_out);

/* all_reduce  proj/src/collectives.cpp:74-88 (rank-ascending fp32 sum). */
int orc_all_reduce(int world, const float* const* inputs, int64_t T, int64_t H, float* out);

/* fused_allreduce_rmsnorm  proj/src/collectives.cpp:134-182 (sequential mode;
 * the reference's parallel mode is bitwise identical).
 * residual_shards[r] is [T_r, H] and is overwritten with r' as in :144. */
int orc_fused_allreduce_rmsnorm(int world, const float* const* inputs, float* const* residual_shards,
                                const int64_t* ranges, const float* weight, int64_t T, int64_t H,
                                float eps, float* output);

/* Wave model  proj/src/wavemodel.cpp:38-49. */
int64_t orc_cta_count(int64_t num_tokens, int64_t tile_tokens, int64_t cta_columns);
int64_t orc_wave_count(int64_t ctas, int64_t sms_available);

/* smart_offset_analytic  proj/src/splitter.cpp:16-53. */
int64_t orc_smart_offset_analytic(int64_t num_tokens, int64_t num_sms, int64_t tile_tokens,
                                  int64_t cta_columns);

/* make_split_plan  proj/src/splitter.cpp:71-88.  out4 = {prefix, suffix, offset, mode}
 * with mode 0 NoSplit, 1 FusedOnly, 2 Overlap. */
int orc_make_split_plan(int64_t num_tokens, int64_t threshold, int64_t num_sms,
                        int64_t tile_tokens, int64_t cta_columns, int64_t* out4);

/* place_sequence_boundaries  proj/src/splitter.cpp:90-105. */
int orc_place_sequence_boundaries(const int64_t* lengths, int n, int64_t total_tokens,
                                  int64_t prefix_tokens, int64_t* prefix_len_out);

/* form_batches  proj/src/workloads.cpp:68-109 (FCFS chunked prefill,
 * decode first).  Requests: prompt[n], output[n], arrival[n] (id = index).
 * out4 rows {total_tokens, decode_token_count, kv_context, num_slices};
 * slices3 rows {request_id, start, len}.  counts = {batches, slices} (always
 * set).  Returns 0, 3 (chunk_size < 1) or 1 (arrays too small). */
int orc_form_batches(const int64_t* prompt, const int64_t* output, const double* arrival, int64_t n,
                     int64_t chunk_size, int64_t* out4, int64_t max_batches, int64_t* slices3,
                     int64_t max_slices, int64_t* counts);

/* bf16 round-to-nearest-even helpers (the GPU's storage format). */
void orc_round_to_bf16(const float* in, float* out, int64_t n);
void orc_f32_to_bf16_bits(const float* in, uint16_t* out, int64_t n);
void orc_bf16_bits_to_f32(const uint16_t* in, float* out, int64_t n);

#ifdef __cplusplus
}
#endif

#endif
