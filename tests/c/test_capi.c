/* test_capi.c -- the C-ABI from plain C99 (no C++ in the caller): the header
 * compiles as C, the library links with gcc, host-side calls and their error
 * taxonomy work without a GPU.  Built and run by tests/test_capi.py. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "tw/tw.h"
#include "tw/tw_split.h"
#include "tw/tw_weave.h"
#include "tw/tw_workload.h"

static int failures = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      ++failures;                                              \
      printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);       \
    }                                                          \
  } while (0)

int main(void) {
  int64_t r[16];
  EXPECT(tw_abi_version() == TW_ABI_VERSION);
  EXPECT(strstr(tw_version(), "sm_100a") != NULL);
  /* SPEC.md:95-97 */
  EXPECT(tw_token_shard_map(10, 4, r) == TW_OK);
  EXPECT(r[0] == 0 && r[1] == 3 && r[2] == 3 && r[3] == 6 && r[4] == 6 && r[5] == 8 && r[6] == 8 && r[7] == 10);
  EXPECT(tw_token_shard_map(16, 1, r) == TW_ERR_CONFIG);
  EXPECT(tw_token_shard_map(-1, 4, r) == TW_ERR_DIMENSION);
  r[2] = 2; /* overlap */
  EXPECT(tw_shard_map_validate(r, 4, 10) == TW_ERR_CONTRACT);
  EXPECT(strlen(tw_last_error()) > 0);
  /* host-side validation precedes device work */
  EXPECT(tw_rmsnorm_residual(NULL, NULL, NULL, NULL, NULL, 4, 8, -1.0f, TW_BF16, 0, NULL) == TW_ERR_NUMERIC);
  EXPECT(tw_rmsnorm_residual(NULL, NULL, NULL, NULL, NULL, 0, 8, 1e-5f, TW_BF16, 0, NULL) == TW_OK);
  /* the planner (B200, dense threshold 1024) */
  {
    int64_t a, b, off;
    int mode;
    EXPECT(tw_make_split_plan(4096, 148, 128, 32, 1024, &a, &b, &off, &mode) == TW_OK);
    EXPECT(a == 1152 && b == 2944 && off == -896 && mode == 2);
    EXPECT(tw_make_split_plan(512, 148, 128, 32, 1024, &a, &b, &off, &mode) == TW_OK && mode == 1);
  }
  /* batch formation (proj/tests/test_workloads.cpp:108-119) */
  {
    tw_request req[1];
    tw_iteration_batch b[8];
    tw_prefill_slice sl[8];
    int64_t nb = 0, ns = 0;
    EXPECT(tw_synth_trace(1, 300, 3, req) == TW_OK);
    EXPECT(tw_form_batches(req, 1, 100, b, 2, sl, 8, &nb, &ns) == TW_ERR_DIMENSION && nb == 6 && ns == 3);
    EXPECT(tw_form_batches(req, 1, 100, b, 8, sl, 8, &nb, &ns) == TW_OK && nb == 6);
    EXPECT(b[0].kv_context == 0 && b[3].kv_context == 300 && b[5].kv_context == 302 && b[5].num_slices == 0);
    EXPECT(sl[2].start == 200 && sl[2].len == 100);
    EXPECT(tw_form_batches(req, 1, 0, b, 8, sl, 8, &nb, &ns) == TW_ERR_CONFIG);
    EXPECT(tw_load_trace("/nonexistent/trace.jsonl", NULL, 0, &nb) == TW_ERR_PARSE);
    EXPECT(strstr(tw_workload_last_error(), "cannot open") != NULL);
  }
  printf("c-abi: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
