// weavesim_dropin.cpp -- the reference's C++ operator API (namespace weavesim)
// re-implemented over the tw C-ABI (include/tw/tw.h).  Host-side validation
// follows the reference exactly (same checks, same order, same exception
// types); the arithmetic runs on the GPU in hand-written sm_100a kernels:
//   rmsnorm_residual         -> tw_rmsnorm_residual (K2)
//   fused_allreduce_rmsnorm  -> tw_fused_allreduce_rmsnorm_group (K1)
//   all_reduce/reduce_scatter-> tw_allreduce_group (K3)
// There is no CPU compute fallback: without a GPU these throw DeviceError.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "tw/tw.h"
#include "weavesim/collectives.hpp"
#include "weavesim/errors.hpp"
#include "weavesim/numerics.hpp"

namespace weavesim {

namespace {

// result matrices at least this large are value-initialised on helper threads
// overlapped with the transfers (rmsnorm_residual below)
constexpr size_t kOverlapFillBytes = 16u << 20;

// A fresh result matrix (TokenMatrix::zeros in the reference) whose
// value-initialisation runs on a helper thread while the caller stages the
// inputs and the kernels run; wait() before the results are copied in.  The
// storage is allocated on the calling thread (glibc's main arena).
class ZerosBehind {
 public:
  ZerosBehind(TokenMatrix& m, std::int64_t T, std::int64_t H) : m_(m) {
    const size_t n = static_cast<size_t>(T * H);
    m.num_tokens = T;
    m.hidden = H;
    if (n * sizeof(float) < kOverlapFillBytes) {
      m.values.assign(n, 0.0f);
      return;
    }
    m.values.reserve(n);
    t_ = std::thread([this, n] { m_.values.resize(n); });
  }
  void wait() {
    if (t_.joinable()) t_.join();
  }
  ~ZerosBehind() { wait(); }  // exception paths: never leave the thread running

 private:
  TokenMatrix& m_;
  std::thread t_;
};

[[noreturn]] void throw_status(tw_status st, const std::string& where) {
  const std::string msg = where + ": " + tw_last_error();
  switch (st) {
    case TW_ERR_DIMENSION: throw DimensionError(msg);
    case TW_ERR_NUMERIC: throw NumericError(msg);
    case TW_ERR_CONFIG: throw ConfigError(msg);
    case TW_ERR_CONTRACT: throw ContractError(msg);
    default: throw DeviceError(msg);
  }
}

void check(tw_status st, const char* where) {
  if (st != TW_OK) throw_status(st, where);
}

// Device scratch buffer owned by the drop-in (grown on demand).
struct DevBuf {
  int device = 0;
  void* ptr = nullptr;
  size_t bytes = 0;
  void reserve(int dev, size_t n) {
    if (ptr && device == dev && bytes >= n) return;
    release();
    device = dev;
    check(tw_device_alloc(dev, std::max<size_t>(n, 256), &ptr), "device_alloc");
    bytes = std::max<size_t>(n, 256);
  }
  void release() {
    if (ptr) tw_device_free(device, ptr);
    ptr = nullptr;
    bytes = 0;
  }
  // No destructor: scratch lives until process exit (the CUDA runtime may
  // already be torn down when static destructors run).
};

int device_count_or_throw() {
  const int n = tw_device_count();
  if (n < 1) throw DeviceError("weavesim (B200 build): no CUDA device visible");
  return n;
}

// Host matrices <-> device: staged through libtw's pinned ring by its host
// thread pool (tw_memcpy_*_staged), not the driver's serial pageable staging.
// scan = TokenMatrix::validate's NaN/Inf check riding on the copy; returns true
// if a non-finite value was found.
bool h2d(void* dst, const std::vector<float>& src, bool scan, const char* where) {
  int nonfinite = 0;
  check(tw_memcpy_h2d_staged(dst, src.data(), src.size() * sizeof(float), TW_F32, scan ? TW_HOST_CHECK_FINITE : 0u,
                             &nonfinite),
        where);
  return nonfinite != 0;
}
void d2h(float* dst, const void* src, size_t bytes, const char* where) {
  check(tw_memcpy_d2h_staged(dst, src, bytes), where);
}

// Cached communicator + per-rank scratch for the RankGroup API.
struct GroupContext {
  tw_comm_t comm = nullptr;
  int world = 0;
  size_t bytes = 0;
  std::vector<int> devices;
  std::vector<DevBuf> residual, weight;
  void release() {
    if (comm) tw_comm_destroy(comm);
    comm = nullptr;
    for (DevBuf& b : residual) b.release();
    for (DevBuf& b : weight) b.release();
  }
};

std::mutex g_mu;
GroupContext* g_ctx = nullptr;  // intentionally never destroyed at exit (see DevBuf)

tw_transport dropin_transport() {
  const char* t = std::getenv("TW_DROPIN_TRANSPORT");
  if (t && std::strcmp(t, "nvls") == 0) return TW_TRANSPORT_NVLS;
  if (t && std::strcmp(t, "auto") == 0) return TW_TRANSPORT_AUTO;
  return TW_TRANSPORT_PEER;  // deterministic rank-ascending fp32 reduction
}

GroupContext& context_for(int world, size_t bytes) {
  if (g_ctx && g_ctx->world == world && g_ctx->bytes >= bytes) return *g_ctx;
  if (g_ctx) {
    g_ctx->release();
    delete g_ctx;
    g_ctx = nullptr;
  }
  auto ctx = std::make_unique<GroupContext>();
  const int ndev = device_count_or_throw();
  ctx->world = world;
  ctx->bytes = std::max<size_t>(bytes, 1 << 20);
  ctx->devices.assign(world, 0);
  if (ndev >= world && world <= 8) {
    for (int r = 0; r < world; ++r) ctx->devices[r] = r;
  }
  tw_status st = tw_comm_create(world, ctx->devices.data(), ctx->bytes, dropin_transport(), &ctx->comm);
  if (st != TW_OK && ndev >= world) {
    // distinct GPUs without peer access: co-locate every rank on GPU 0
    ctx->devices.assign(world, 0);
    st = tw_comm_create(world, ctx->devices.data(), ctx->bytes, TW_TRANSPORT_PEER, &ctx->comm);
  }
  check(st, "fused_allreduce_rmsnorm: communicator");
  ctx->residual.resize(world);
  ctx->weight.resize(world);
  g_ctx = ctx.release();
  return *g_ctx;
}

}  // namespace

// ---- numerics (proj/src/numerics.cpp) ----------------------------------------------

TokenMatrix TokenMatrix::zeros(std::int64_t tokens, std::int64_t hidden) {
  TokenMatrix m;
  m.num_tokens = tokens;
  m.hidden = hidden;
  if (tokens < 0 || hidden < 1) throw DimensionError("TokenMatrix requires T >= 0 and H >= 1");
  m.values.assign(static_cast<size_t>(tokens * hidden), 0.0f);
  return m;
}

void TokenMatrix::validate() const {
  if (num_tokens < 0 || hidden < 1) throw DimensionError("TokenMatrix requires T >= 0 and H >= 1");
  if (values.size() != static_cast<size_t>(num_tokens * hidden))
    throw DimensionError("TokenMatrix values length must equal T*H");
  for (float v : values)
    if (!std::isfinite(v)) throw NumericError("TokenMatrix contains NaN/Inf");
}

NormResult rmsnorm_residual(const TokenMatrix& input, const TokenMatrix& residual, const NormParams& params) {
  // Validation in the reference's order (numerics.cpp:30-49).  When the shapes,
  // weight and epsilon are consistent the NaN/Inf scans of input and residual
  // ride on the pipeline's staging copy (TW_HOST_CHECK_FINITE, same exception
  // type and message); any structural problem takes the reference's serial
  // order so the first exception thrown is the reference's.
  auto structural_ok = [](const TokenMatrix& m) {
    return m.num_tokens >= 0 && m.hidden >= 1 && m.values.size() == static_cast<size_t>(m.num_tokens * m.hidden);
  };
  const bool fast = structural_ok(input) && structural_ok(residual) && input.same_shape(residual) &&
                    static_cast<std::int64_t>(params.weight.size()) == input.hidden &&
                    (params.epsilon > 0.0f || params.epsilon == 0.0f);
  if (!fast) {
    input.validate();
    residual.validate();
    if (!input.same_shape(residual)) throw DimensionError("rmsnorm_residual: input and residual shapes differ");
    if (static_cast<std::int64_t>(params.weight.size()) != input.hidden)
      throw DimensionError("rmsnorm_residual: weight length must equal hidden size");
    throw NumericError("rmsnorm_residual: epsilon must be nonnegative");
  }
  const std::int64_t T = input.num_tokens, H = input.hidden;
  NormResult result;
  const size_t n = static_cast<size_t>(T * H);
  if (n * sizeof(float) < kOverlapFillBytes) {
    result.output = TokenMatrix::zeros(T, H);
    result.residual_out = TokenMatrix::zeros(T, H);
    if (T == 0) return result;
    device_count_or_throw();
    std::lock_guard<std::mutex> lock(g_mu);
    // Host matrices in, host matrices out: pinned-ring staging by host threads
    // around the chunked H2D | K2 | D2H pipeline.
    const tw_status st = tw_rmsnorm_residual_host_sync(input.values.data(), residual.values.data(),
                                                       result.residual_out.values.data(), result.output.values.data(),
                                                       params.weight.data(), T, H, params.epsilon, TW_F32,
                                                       TW_HOST_CHECK_FINITE);
    if (st == TW_ERR_NUMERIC) throw NumericError("TokenMatrix contains NaN/Inf");
    check(st, "rmsnorm_residual");
    return result;
  }
  device_count_or_throw();
  // The two fresh result matrices (TokenMatrix::zeros in the reference) are
  // allocated here, on the calling thread -- a second thread would allocate
  // from its own glibc arena, measured 5x slower for 256 MiB blocks -- and
  // value-initialised by two helper threads in ~4 MiB steps while the
  // pipeline stages, transfers and computes (2 x ~18 ms of single-thread
  // zero-fill at 8192 x 8192 that used to precede it).  resize() within the
  // reserved capacity never reallocates, so the row pointers taken below
  // stay valid; the pipeline copies chunk k's results in only once both
  // fills have published rows past it (tw_rmsnorm_residual_host_sync_gated).
  for (TokenMatrix* m : {&result.output, &result.residual_out}) {
    m->num_tokens = T;
    m->hidden = H;
    m->values.reserve(n);
  }
  float* out = result.output.values.data();
  float* res_out = result.residual_out.values.data();
  alignas(64) std::int64_t ready[2] = {0, 0};
  std::atomic<bool> stop{false};
  const std::int64_t step = std::max<std::int64_t>(1, static_cast<std::int64_t>((4u << 20) / (H * sizeof(float))));
  auto fill = [&](std::vector<float>* v, std::int64_t* rows) {
    for (std::int64_t t = 0; t < T && !stop.load(std::memory_order_relaxed);) {
      t = std::min(T, t + step);
      v->resize(static_cast<size_t>(t * H));
      __atomic_store_n(rows, t, __ATOMIC_RELEASE);
    }
  };
  std::thread f0(fill, &result.output.values, &ready[0]);
  std::thread f1(fill, &result.residual_out.values, &ready[1]);
  tw_status st;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    st = tw_rmsnorm_residual_host_sync_gated(input.values.data(), residual.values.data(), res_out, out,
                                             params.weight.data(), T, H, params.epsilon, TW_F32,
                                             TW_HOST_CHECK_FINITE, ready, 2);
  }
  if (st != TW_OK) stop.store(true, std::memory_order_relaxed);
  f0.join();
  f1.join();
  if (st == TW_ERR_NUMERIC) throw NumericError("TokenMatrix contains NaN/Inf");
  check(st, "rmsnorm_residual");
  return result;
}

// ---- collectives (proj/src/collectives.cpp) -----------------------------------------

std::int64_t ShardMap::total_tokens() const { return ranges.empty() ? 0 : ranges.back().end; }

void ShardMap::validate(std::int64_t total) const {
  std::vector<std::int64_t> flat;
  for (const TokenRange& r : ranges) {
    flat.push_back(r.begin);
    flat.push_back(r.end);
  }
  const tw_status st = tw_shard_map_validate(flat.empty() ? nullptr : flat.data(), world_size(), total);
  if (st != TW_OK) throw ContractError(std::string("ShardMap: ") + tw_last_error());
}

ShardMap token_shard_map(std::int64_t num_tokens, int world_size) {
  if (world_size < 2) throw ConfigError("token_shard_map: world_size must be >= 2");
  if (num_tokens < 0) throw DimensionError("token_shard_map: negative token count");
  std::vector<std::int64_t> flat(2 * static_cast<size_t>(world_size));
  check(tw_token_shard_map(num_tokens, world_size, flat.data()), "token_shard_map");
  ShardMap m;
  for (int r = 0; r < world_size; ++r) m.ranges.push_back({flat[2 * r], flat[2 * r + 1]});
  return m;
}

void RankGroup::validate() const {
  if (world_size < 2) throw ConfigError("RankGroup: world_size must be >= 2");
  if (static_cast<int>(inputs.size()) != world_size)
    throw DimensionError("RankGroup: one input buffer per rank required");
  for (const TokenMatrix& m : inputs) {
    m.validate();
    if (!m.same_shape(inputs[0])) throw DimensionError("RankGroup: per-rank input shapes differ");
  }
}

void RankGroup::validate_residual(const ShardMap& shards) const {
  shards.validate(num_tokens());
  if (shards.world_size() != world_size) throw ContractError("RankGroup: shard map world size mismatch");
  if (static_cast<int>(residual_shards.size()) != world_size)
    throw DimensionError("RankGroup: one residual shard per rank required");
  for (int r = 0; r < world_size; ++r) {
    residual_shards[r].validate();
    if (residual_shards[r].num_tokens != shards.ranges[r].size() || residual_shards[r].hidden != hidden())
      throw DimensionError("RankGroup: residual shard shape does not match shard map");
  }
}

namespace {

// Upload the group's inputs into the communicator's symmetric INPUT buffers.
// scan: the inputs' NaN/Inf check rides on the copies (NumericError, the
// reference's message, before anything user-visible is written).
void upload_inputs(GroupContext& ctx, const RankGroup& group, bool scan = false) {
  bool nonfinite = false;
  for (int r = 0; r < group.world_size; ++r) {
    void* dst = nullptr;
    check(tw_comm_buffer(ctx.comm, r, TW_BUF_INPUT, &dst), "comm_buffer");
    nonfinite |= h2d(dst, group.inputs[r].values, scan, "H2D inputs");
  }
  if (nonfinite) throw NumericError("TokenMatrix contains NaN/Inf");
}

// The reference's validation of fused_allreduce_rmsnorm (collectives.cpp:41-69,
// 157-163) WITHOUT its NaN/Inf scans: true when only a non-finite value could
// still make it throw, so the scans can ride on the staging copies (same
// exception, same message).  Anything else takes the reference's serial order.
bool fused_structurally_ok(const RankGroup& g, const NormParams& params, const ShardMap& shards) {
  auto ok = [](const TokenMatrix& m) {
    return m.num_tokens >= 0 && m.hidden >= 1 && m.values.size() == static_cast<size_t>(m.num_tokens * m.hidden);
  };
  if (g.world_size < 2 || static_cast<int>(g.inputs.size()) != g.world_size) return false;
  for (const TokenMatrix& m : g.inputs)
    if (!ok(m) || !m.same_shape(g.inputs[0])) return false;
  try {
    shards.validate(g.num_tokens());
  } catch (...) {
    return false;
  }
  if (shards.world_size() != g.world_size || static_cast<int>(g.residual_shards.size()) != g.world_size) return false;
  for (int r = 0; r < g.world_size; ++r) {
    const TokenMatrix& m = g.residual_shards[r];
    if (!ok(m) || m.num_tokens != shards.ranges[r].size() || m.hidden != g.hidden()) return false;
  }
  return static_cast<std::int64_t>(params.weight.size()) == g.hidden();
}

// RankGroups wider than a communicator (TW_MAX_RANKS): the rank-ascending
// fp32 sum as a chain of K2 launches on device 0 -- K2's residual_out is
// x + res in fp32, so acc <- in[r] + acc reproduces reduce_element's
// ((0 + in[0]) + in[1]) + ... bit for bit (fp32 addition commutes; 0 + x = x).
// Returns the device buffer holding the sum (scratch owned here).
struct WideScratch {
  DevBuf in, acc, tmp, out, weight;
};
WideScratch g_wide;  // guarded by g_mu

void* chain_sum_on_device(const RankGroup& group) {
  const std::int64_t T = group.num_tokens(), H = group.hidden();
  const size_t nb = static_cast<size_t>(T * H) * sizeof(float);
  WideScratch& w = g_wide;
  for (DevBuf* b : {&w.in, &w.acc, &w.tmp, &w.out}) b->reserve(0, nb);
  w.weight.reserve(0, static_cast<size_t>(H) * sizeof(float));
  const std::vector<float> ones(static_cast<size_t>(H), 1.0f);
  check(tw_memcpy(w.weight.ptr, ones.data(), ones.size() * sizeof(float), nullptr), "H2D weight");
  h2d(w.acc.ptr, group.inputs[0].values, false, "H2D input");  // 0 + in[0] == in[0]
  for (int r = 1; r < group.world_size; ++r) {
    h2d(w.in.ptr, group.inputs[r].values, false, "H2D input");
    check(tw_rmsnorm_residual(w.in.ptr, w.acc.ptr, w.tmp.ptr, w.out.ptr, static_cast<const float*>(w.weight.ptr), T,
                              H, 0.0f, TW_F32, 0, nullptr),
          "rank-order sum");
    std::swap(w.acc.ptr, w.tmp.ptr);
  }
  check(tw_device_synchronize(0), "rank-order sum");
  return w.acc.ptr;
}

// scan: the inputs' NaN/Inf check of RankGroup::validate rides on the upload
// (the caller has checked everything else, in the reference's order).
TokenMatrix reduce_on_device(const RankGroup& group, bool scan = false) {
  const std::int64_t T = group.num_tokens(), H = group.hidden();
  TokenMatrix out;
  if (T == 0) return TokenMatrix::zeros(T, H);
  ZerosBehind zeros(out, T, H);
  const size_t nb = static_cast<size_t>(T * H) * sizeof(float);
  if (group.world_size > TW_MAX_RANKS) {
    void* sum = chain_sum_on_device(group);
    zeros.wait();
    d2h(out.values.data(), sum, nb, "D2H all_reduce");
    return out;
  }
  GroupContext& ctx = context_for(group.world_size, nb);
  upload_inputs(ctx, group, scan);
  check(tw_allreduce_group(ctx.comm, T, H, 0, TW_F32, 8, nullptr), "all_reduce");
  for (int d : ctx.devices) check(tw_device_synchronize(d), "all_reduce");
  check(tw_comm_check(ctx.comm), "all_reduce");
  void* src = nullptr;
  check(tw_comm_buffer(ctx.comm, 0, TW_BUF_OUTPUT, &src), "comm_buffer");
  zeros.wait();
  d2h(out.values.data(), src, nb, "D2H all_reduce");
  return out;
}

// RankGroup::validate without its NaN/Inf scans (collectives.cpp:41-50): when
// true, the scans ride on the staged upload (same exception and message).
bool inputs_structurally_ok(const RankGroup& g) {
  if (g.world_size < 2 || static_cast<int>(g.inputs.size()) != g.world_size || g.world_size > TW_MAX_RANKS ||
      tw_device_count() < 1)
    return false;
  for (const TokenMatrix& m : g.inputs)
    if (m.num_tokens < 0 || m.hidden < 1 || m.values.size() != static_cast<size_t>(m.num_tokens * m.hidden) ||
        !m.same_shape(g.inputs[0]))
      return false;
  return true;
}

}  // namespace

TokenMatrix all_reduce(const RankGroup& group) {
  const bool fast = inputs_structurally_ok(group);
  if (!fast) group.validate();
  std::lock_guard<std::mutex> lock(g_mu);
  return reduce_on_device(group, fast);
}

std::vector<TokenMatrix> reduce_scatter(const RankGroup& group, const ShardMap& shards) {
  // the reference validates the group (NaN/Inf included) BEFORE the shard map:
  // the scan may ride on the upload only when the shard map is valid too
  bool fast = inputs_structurally_ok(group);
  if (fast) {
    try {
      shards.validate(group.num_tokens());
    } catch (...) {
      fast = false;
    }
  }
  if (!fast) {
    group.validate();
    shards.validate(group.num_tokens());
  }
  TokenMatrix sum;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    sum = reduce_on_device(group, fast);
  }
  const std::int64_t H = group.hidden();
  std::vector<TokenMatrix> out;
  for (const TokenRange& range : shards.ranges) {
    TokenMatrix shard = TokenMatrix::zeros(range.size(), H);
    std::copy(sum.values.begin() + range.begin * H, sum.values.begin() + range.end * H, shard.values.begin());
    out.push_back(std::move(shard));
  }
  return out;
}

TokenMatrix all_gather(const std::vector<TokenMatrix>& per_rank_shards, const ShardMap& shards) {
  if (per_rank_shards.size() != shards.ranges.size())
    throw DimensionError("all_gather: shard count does not match shard map");
  const std::int64_t total = shards.total_tokens();
  shards.validate(total);
  const std::int64_t H = per_rank_shards.empty() ? 1 : per_rank_shards[0].hidden;
  TokenMatrix out = TokenMatrix::zeros(total, H);
  for (size_t r = 0; r < per_rank_shards.size(); ++r) {
    const TokenRange& range = shards.ranges[r];
    const TokenMatrix& shard = per_rank_shards[r];
    if (shard.num_tokens != range.size() || shard.hidden != H)
      throw DimensionError("all_gather: shard shape does not match its range");
    std::copy(shard.values.begin(), shard.values.end(), out.values.begin() + range.begin * H);
  }
  return out;
}

TokenMatrix fused_allreduce_rmsnorm(RankGroup& group, const NormParams& params, const ShardMap& shards,
                                    bool /*parallel*/) {
  // The reference's checks in its order; when the structure is sound the
  // NaN/Inf scans of the inputs and shards ride on the staging copies below.
  // (no GPU visible: the serial order, so a NaN is still a NumericError, not a DeviceError)
  const bool fast =
      fused_structurally_ok(group, params, shards) && group.world_size <= TW_MAX_RANKS && tw_device_count() > 0;
  if (!fast) {
    group.validate();
    group.validate_residual(shards);
    if (static_cast<std::int64_t>(params.weight.size()) != group.hidden())
      throw DimensionError("fused_allreduce_rmsnorm: weight length must equal hidden size");
  }
  const std::int64_t T = group.num_tokens(), H = group.hidden();
  if (T == 0) return TokenMatrix::zeros(T, H);
  const int W = group.world_size;
  const size_t nb = static_cast<size_t>(T * H) * sizeof(float);
  TokenMatrix output;
  ZerosBehind zeros(output, T, H);
  std::lock_guard<std::mutex> lock(g_mu);
  if (W > TW_MAX_RANKS) {
    // wider than a communicator: the chained rank-order sum, then one K2 over
    // all T rows with the shards' residual rows (r' = v + res, the same fp32
    // and double arithmetic as fused_rank_body, collectives.cpp:134-153)
    void* sum = chain_sum_on_device(group);
    WideScratch& w = g_wide;
    std::vector<float> res(static_cast<size_t>(T * H));
    for (int r = 0; r < W; ++r)
      std::copy(group.residual_shards[r].values.begin(), group.residual_shards[r].values.end(),
                res.begin() + shards.ranges[r].begin * H);
    h2d(w.in.ptr, res, false, "H2D residual");
    check(tw_memcpy(w.weight.ptr, params.weight.data(), static_cast<size_t>(H) * sizeof(float), nullptr),
          "H2D weight");
    check(tw_rmsnorm_residual(sum, w.in.ptr, w.tmp.ptr, w.out.ptr, static_cast<const float*>(w.weight.ptr), T, H,
                              params.epsilon, TW_F32, 0, nullptr),
          "fused_allreduce_rmsnorm");
    check(tw_device_synchronize(0), "fused_allreduce_rmsnorm");
    zeros.wait();
    d2h(output.values.data(), w.out.ptr, nb, "D2H output");
    d2h(res.data(), w.tmp.ptr, nb, "D2H residual");
    for (int r = 0; r < W; ++r)
      std::copy(res.begin() + shards.ranges[r].begin * H, res.begin() + shards.ranges[r].end * H,
                group.residual_shards[r].values.begin());
    return output;
  }
  GroupContext& ctx = context_for(W, nb);
  upload_inputs(ctx, group, fast);
  std::vector<void*> res(W, nullptr);
  std::vector<const float*> wts(W, nullptr);
  std::vector<std::int64_t> flat;
  for (int r = 0; r < W; ++r) {
    const size_t rb = group.residual_shards[r].values.size() * sizeof(float);
    ctx.residual[r].reserve(ctx.devices[r], rb);
    ctx.weight[r].reserve(ctx.devices[r], H * sizeof(float));
    if (h2d(ctx.residual[r].ptr, group.residual_shards[r].values, fast, "H2D residual"))
      throw NumericError("TokenMatrix contains NaN/Inf");
    check(tw_memcpy(ctx.weight[r].ptr, params.weight.data(), H * sizeof(float), nullptr), "H2D weight");
    res[r] = rb ? ctx.residual[r].ptr : nullptr;
    wts[r] = static_cast<const float*>(ctx.weight[r].ptr);
    flat.push_back(shards.ranges[r].begin);
    flat.push_back(shards.ranges[r].end);
  }
  check(tw_fused_allreduce_rmsnorm_group(ctx.comm, T, H, 0, flat.data(), res.data(), wts.data(), params.epsilon, TW_F32,
                                         8, 0u, nullptr),
        "fused_allreduce_rmsnorm");
  for (int d : ctx.devices) check(tw_device_synchronize(d), "fused_allreduce_rmsnorm");
  check(tw_comm_check(ctx.comm), "fused_allreduce_rmsnorm");
  void* src = nullptr;
  check(tw_comm_buffer(ctx.comm, 0, TW_BUF_OUTPUT, &src), "comm_buffer");
  zeros.wait();
  d2h(output.values.data(), src, nb, "D2H output");
  for (int r = 0; r < W; ++r) {
    const size_t rb = group.residual_shards[r].values.size() * sizeof(float);
    d2h(group.residual_shards[r].values.data(), ctx.residual[r].ptr, rb, "D2H residual");
  }
  return output;
}

}  // namespace weavesim
