/*
 * tw_workload.h -- C-ABI of request traces and chunked-prefill batch
 * formation (libweavesim_b200.so; the C++ API is include/weavesim/workloads.hpp).
 * Same semantics and error taxonomy as the reference
 * (proj/include/weavesim/workloads.hpp:10-52, proj/src/workloads.cpp:14-109).
 * The measured throughput run over these batches is tw_weave_throughput
 * (include/tw/tw_weave.h).
 */
#ifndef TW_TW_WORKLOAD_H
#define TW_TW_WORKLOAD_H

#include "tw/tw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* weavesim::Request (workloads.hpp:12-17). */
typedef struct tw_request {
  int64_t id;
  int64_t prompt_tokens;
  int64_t output_tokens;
  double arrival_s;
} tw_request;

/* weavesim::PrefillSlice (workloads.hpp:26-30). */
typedef struct tw_prefill_slice {
  int64_t request_id;
  int64_t start;
  int64_t len;
} tw_prefill_slice;

/* weavesim::IterationBatch (workloads.hpp:32-39); its prefill slices are
 * slices[first_slice .. first_slice + num_slices) of the flat slice array. */
typedef struct tw_iteration_batch {
  int64_t total_tokens;
  int64_t decode_token_count;
  int64_t kv_context;
  int64_t first_slice;
  int64_t num_slices;
} tw_iteration_batch;

/* Message of the last failing call of this header on this thread. */
TW_API const char* tw_workload_last_error(void);

/* synth_trace: `count` identical requests into out[count] (CONFIG on bad args). */
TW_API tw_status tw_synth_trace(int64_t count, int64_t prompt_len, int64_t output_len, tw_request* out);

/* load_trace: *count = requests in the file; up to `capacity` are written to
 * out (out may be NULL with capacity 0 to size the array).  PARSE on a
 * missing file, bad JSON (message names the line) or out-of-range values. */
TW_API tw_status tw_load_trace(const char* path, tw_request* out, int64_t capacity, int64_t* count);
TW_API tw_status tw_save_trace(const tw_request* requests, int64_t n, const char* path);

/* form_batches: writes up to max_batches batches and max_slices slices and
 * sets *n_batches / *n_slices to the totals.  If either array is too small the
 * call returns DIMENSION with the totals set (call again with larger arrays).
 * chunk_size < 1 -> CONFIG. */
TW_API tw_status tw_form_batches(const tw_request* requests, int64_t n, int64_t chunk_size,
                                 tw_iteration_batch* batches, int64_t max_batches, tw_prefill_slice* slices,
                                 int64_t max_slices, int64_t* n_batches, int64_t* n_slices);

#ifdef __cplusplus
}
#endif

#endif
