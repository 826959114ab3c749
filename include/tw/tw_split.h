/*
 * tw_split.h -- C-ABI of the weave's token-split planner (libweavesim_b200.so;
 * the C++ API is include/weavesim/splitter.hpp).  Same semantics and error
 * taxonomy as the reference planner (proj/src/splitter.cpp:11-105).
 */
#ifndef TW_TW_SPLIT_H
#define TW_TW_SPLIT_H

#include "tw/tw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* mode: 0 NoSplit, 1 FusedOnly, 2 Overlap (SplitMode, splitter.hpp:11). */
TW_API tw_status tw_make_split_plan(int64_t num_tokens, int num_sms, int tile_tokens, int cta_columns,
                                    int64_t threshold_tokens, int64_t* prefix, int64_t* suffix, int64_t* offset,
                                    int* mode);
TW_API tw_status tw_smart_offset_analytic(int64_t num_tokens, int num_sms, int tile_tokens, int cta_columns,
                                          int64_t* offset);
/* Alg. 1 over offset_grid[n]: forward(prefix, suffix, ctx) returns a time. */
TW_API tw_status tw_smart_offset_sweep(int64_t num_tokens, const int64_t* offset_grid, int n,
                                       double (*forward)(int64_t, int64_t, void*), void* ctx, int64_t* offset);
TW_API tw_status tw_place_sequence_boundaries(const int64_t* lengths, int n, int64_t total_tokens,
                                              int64_t prefix_tokens, int64_t* prefix_len_out);

#ifdef __cplusplus
}
#endif

#endif
