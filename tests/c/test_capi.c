/* test_capi.c -- the C-ABI from plain C99 (no C++ in the caller): the header
 * compiles as C, the library links with gcc, host-side calls and their error
 * taxonomy work without a GPU.  Built and run by tests/test_capi.py. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "tw/tw.h"
#include "tw/tw_split.h"
#include "tw/tw_weave.h"

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
  printf("c-abi: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
