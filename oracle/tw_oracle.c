/*
 * tw_oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY (see tw_oracle.h): the checker, never the product.
 *
 * Parity pinned against oracle/_ref/libweavesim_ref.so (the reference's own
 * proj/src/{numerics,collectives,wavemodel,splitter,workloads}.cpp compiled unmodified,
 * see oracle/Makefile) and against tests/golden/ fixtures generated from it by
 * tests/golden/make_golden.py.  Compile with -ffp-contract=off so the float
 * expression order matches the reference build (no FMA contraction).
 */
#include "tw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* proj/src/collectives.cpp:26-39 */
int orc_token_shard_map(int64_t num_tokens, int world, int64_t* ranges) {
  if (world < 2) return ORC_CONFIG;
  if (num_tokens < 0) return ORC_DIMENSION;
  const int64_t base = num_tokens / world;
  const int64_t extra = num_tokens % world;
  int64_t cursor = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t len = base + (r < extra ? 1 : 0);
    ranges[2 * r] = cursor;
    ranges[2 * r + 1] = cursor + len;
    cursor += len;
  }
  return ORC_OK;
}

/* proj/src/collectives.cpp:14-24 */
int orc_shard_map_validate(const int64_t* ranges, int world, int64_t total) {
  if (world < 1) return ORC_CONTRACT;
  int64_t cursor = 0;
  for (int r = 0; r < world; ++r) {
    if (ranges[2 * r] != cursor || ranges[2 * r + 1] < ranges[2 * r]) return ORC_CONTRACT;
    cursor = ranges[2 * r + 1];
  }
  return cursor == total ? ORC_OK : ORC_CONTRACT;
}

/* proj/src/numerics.cpp:25-27 */
int orc_all_finite(const float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(v[i])) return ORC_NUMERIC;
  }
  return ORC_OK;
}

/* One token row: r' = a + b (fp32), ss += double(r')^2 in ascending j, then
 * inv = 1/sqrtf(float(ss/H) + eps), out = (r' * inv) * w.  This is the body
 * shared by proj/src/numerics.cpp:50-62 and proj/src/collectives.cpp:139-152. */
static void norm_row(const float* r_row, const float* weight, int64_t H, float eps, float* out) {
  double sum_sq = 0.0;
  for (int64_t j = 0; j < H; ++j) sum_sq += (double)r_row[j] * (double)r_row[j];
  const float inv_rms = 1.0f / sqrtf((float)(sum_sq / (double)H) + eps);
  for (int64_t j = 0; j < H; ++j) out[j] = r_row[j] * inv_rms * weight[j];
}

/* proj/src/numerics.cpp:30-64 */
int orc_rmsnorm_residual(const float* input, const float* residual, const float* weight,
                         int64_t T, int64_t H, float eps, float* output, float* residual_out) {
  if (T < 0 || H < 1) return ORC_DIMENSION;
  if (orc_all_finite(input, T * H) || orc_all_finite(residual, T * H)) return ORC_NUMERIC;
  if (!(eps > 0.0f) && eps != 0.0f) return ORC_NUMERIC;
  for (int64_t t = 0; t < T; ++t) {
    const float* a = input + t * H;
    const float* b = residual + t * H;
    float* r = residual_out + t * H;
    for (int64_t j = 0; j < H; ++j) r[j] = a[j] + b[j];
    norm_row(r, weight, H, eps, output + t * H);
  }
  return ORC_OK;
}

/* proj/src/collectives.cpp:74-88: acc starts at 0.0f and adds ranks 0..N-1. */
int orc_all_reduce(int world, const float* const* inputs, int64_t T, int64_t H, float* out) {
  if (world < 2) return ORC_CONFIG;
  const int64_t n = T * H;
  for (int r = 0; r < world; ++r) {
    if (orc_all_finite(inputs[r], n)) return ORC_NUMERIC;
  }
  for (int64_t i = 0; i < n; ++i) {
    float acc = 0.0f;
    for (int r = 0; r < world; ++r) acc += inputs[r][i];
    out[i] = acc;
  }
  return ORC_OK;
}

/* proj/src/collectives.cpp:134-182 (validation order :158-163, body :134-153). */
int orc_fused_allreduce_rmsnorm(int world, const float* const* inputs, float* const* residual_shards,
                                const int64_t* ranges, const float* weight, int64_t T, int64_t H,
                                float eps, float* output) {
  if (world < 2) return ORC_CONFIG;
  if (T < 0 || H < 1) return ORC_DIMENSION;
  for (int r = 0; r < world; ++r) {
    if (orc_all_finite(inputs[r], T * H)) return ORC_NUMERIC;
  }
  if (orc_shard_map_validate(ranges, world, T)) return ORC_CONTRACT;
  for (int r = 0; r < world; ++r) {
    const int64_t len = ranges[2 * r + 1] - ranges[2 * r];
    if (orc_all_finite(residual_shards[r], len * H)) return ORC_NUMERIC;
  }
  float* row = (float*)malloc(sizeof(float) * (size_t)(H > 0 ? H : 1));
  if (!row) return ORC_DIMENSION;
  for (int r = 0; r < world; ++r) {
    const int64_t begin = ranges[2 * r];
    const int64_t len = ranges[2 * r + 1] - begin;
    for (int64_t t = 0; t < len; ++t) {
      const int64_t token = begin + t;
      float* res = residual_shards[r] + t * H;
      for (int64_t j = 0; j < H; ++j) {
        float v = 0.0f;
        for (int q = 0; q < world; ++q) v += inputs[q][token * H + j];
        res[j] = v + res[j];
      }
      memcpy(row, res, sizeof(float) * (size_t)H);
      norm_row(row, weight, H, eps, output + token * H);
    }
  }
  free(row);
  return ORC_OK;
}

/* proj/src/wavemodel.cpp:38-43 */
int64_t orc_cta_count(int64_t num_tokens, int64_t tile_tokens, int64_t cta_columns) {
  if (num_tokens <= 0) return 0;
  return ((num_tokens + tile_tokens - 1) / tile_tokens) * cta_columns;
}

/* proj/src/wavemodel.cpp:45-49 */
int64_t orc_wave_count(int64_t ctas, int64_t sms_available) {
  return (ctas + sms_available - 1) / sms_available;
}

/* proj/src/splitter.cpp:16-53 */
int64_t orc_smart_offset_analytic(int64_t num_tokens, int64_t num_sms, int64_t tile_tokens,
                                  int64_t cta_columns) {
  const int64_t half = num_tokens / 2;
  const int64_t all_prefix_offset = num_tokens - half;
  if (orc_wave_count(orc_cta_count(num_tokens, tile_tokens, cta_columns), num_sms) <= 1) {
    return all_prefix_offset;
  }
  const int64_t row_tiles = (num_tokens + tile_tokens - 1) / tile_tokens;
  if (row_tiles < 2) return all_prefix_offset;
  int64_t best_prefix = half;
  int64_t best_waves = INT64_MAX;
  int64_t best_imbalance = INT64_MAX;
  for (int64_t p = 0; p < row_tiles; ++p) {
    /* p == 0 stands for the equal split, considered first (:44). */
    int64_t prefix = p == 0 ? half : p * tile_tokens;
    if (p > 0 && prefix > num_tokens - 1) prefix = num_tokens - 1;
    if (prefix < 1 || prefix >= num_tokens) continue;
    const int64_t waves =
        orc_wave_count(orc_cta_count(prefix, tile_tokens, cta_columns), num_sms) +
        orc_wave_count(orc_cta_count(num_tokens - prefix, tile_tokens, cta_columns), num_sms);
    const int64_t imbalance = llabs(prefix - half);
    if (waves < best_waves || (waves == best_waves && imbalance < best_imbalance)) {
      best_waves = waves;
      best_imbalance = imbalance;
      best_prefix = prefix;
    }
  }
  return best_prefix - half;
}

/* proj/src/splitter.cpp:11-14, 71-88 */
int orc_make_split_plan(int64_t num_tokens, int64_t threshold, int64_t num_sms,
                        int64_t tile_tokens, int64_t cta_columns, int64_t* out4) {
  if (threshold < 1) return ORC_CONFIG;
  if (num_tokens < 0) return ORC_DIMENSION;
  if (num_tokens < threshold) {
    out4[0] = num_tokens;
    out4[1] = 0;
    out4[2] = 0;
    out4[3] = 1;
    return ORC_OK;
  }
  const int64_t half = num_tokens / 2;
  const int64_t offset = orc_smart_offset_analytic(num_tokens, num_sms, tile_tokens, cta_columns);
  out4[0] = half + offset;
  out4[1] = num_tokens - out4[0];
  out4[2] = offset;
  out4[3] = out4[1] == 0 ? 1 : 2;
  return ORC_OK;
}

/* proj/src/splitter.cpp:90-105 */
int orc_place_sequence_boundaries(const int64_t* lengths, int n, int64_t total_tokens,
                                  int64_t prefix_tokens, int64_t* prefix_len_out) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += lengths[i];
  if (total != total_tokens) return ORC_CONTRACT;
  int64_t remaining = prefix_tokens;
  for (int i = 0; i < n; ++i) {
    int64_t take = remaining < 0 ? 0 : remaining;
    if (take > lengths[i]) take = lengths[i];
    prefix_len_out[i] = take;
    remaining -= take;
  }
  return ORC_OK;
}

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

void orc_round_to_bf16(const float* in, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = bf16_to_f32(f32_to_bf16_rne(in[i]));
}

void orc_f32_to_bf16_bits(const float* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = f32_to_bf16_rne(in[i]);
}

void orc_bf16_bits_to_f32(const uint16_t* in, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = bf16_to_f32(in[i]);
}

/* ---- form_batches  proj/src/workloads.cpp:68-109 --------------------------------
 * A literal restatement: every iteration rescans the FCFS order twice (decode
 * pass :86-95, prefill pass :96-107); the stable sort by arrival (:76-80) is an
 * insertion sort (stable, ties keep index order). */
int orc_form_batches(const int64_t* prompt, const int64_t* output, const double* arrival, int64_t n,
                     int64_t chunk_size, int64_t* out4, int64_t max_batches, int64_t* slices3,
                     int64_t max_slices, int64_t* counts) {
  if (chunk_size < 1) return 3;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* prefilled = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  int64_t* decoded = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = i;
    while (j > 0 && (arrival ? arrival[order[j - 1]] : 0.0) > (arrival ? arrival[i] : 0.0)) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = i;
  }
  int64_t nb = 0, ns = 0;
  int overflow = 0;
  for (;;) {
    int64_t decode = 0, kv = 0, total = 0, first = ns, nslice = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t i = order[k];
      if (prefilled[i] == prompt[i] && decoded[i] < output[i]) {
        ++decoded[i];
        ++decode;
        kv += prompt[i] + decoded[i] - 1;
      }
    }
    int64_t budget = chunk_size - decode;
    for (int64_t k = 0; k < n; ++k) {
      if (budget <= 0) break;
      const int64_t i = order[k];
      if (prefilled[i] == prompt[i]) continue;
      const int64_t left = prompt[i] - prefilled[i];
      const int64_t take = budget < left ? budget : left;
      if (ns < max_slices) {
        slices3[3 * ns + 0] = i;
        slices3[3 * ns + 1] = prefilled[i];
        slices3[3 * ns + 2] = take;
      } else {
        overflow = 1;
      }
      ++ns;
      ++nslice;
      kv += prefilled[i];
      prefilled[i] += take;
      budget -= take;
      total += take;
    }
    total += decode;
    if (total == 0) {
      ns = first;
      break;
    }
    if (nb < max_batches) {
      out4[4 * nb + 0] = total;
      out4[4 * nb + 1] = decode;
      out4[4 * nb + 2] = kv;
      out4[4 * nb + 3] = nslice;
    } else {
      overflow = 1;
    }
    ++nb;
  }
  counts[0] = nb;
  counts[1] = ns;
  free(order);
  free(prefilled);
  free(decoded);
  return overflow ? 1 : 0;
}
