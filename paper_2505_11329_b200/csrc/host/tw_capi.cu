// tw_capi.cu -- the C-ABI (include/tw/tw.h): argument validation with the
// reference's error taxonomy, the communicator (NVLS multicast objects or
// peer buffers, signal pads), and dispatch to the row engine.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../kernels/tw_launch.h"
#include "tw_internal.h"

namespace tw {

namespace {
// POD storage: safe to touch from static destructors of other libraries
// (a thread_local std::string may already be destroyed at process exit).
thread_local char g_last_error[1024];
}

void set_error(const std::string& msg) {
  const size_t n = std::min(msg.size(), sizeof(g_last_error) - 1);
  std::memcpy(g_last_error, msg.data(), n);
  g_last_error[n] = '\0';
}
void clear_error() { g_last_error[0] = '\0'; }

tw_status fail(tw_status code, const std::string& msg) {
  set_error(msg);
  return code;
}

tw_status cuda_fail(cudaError_t e, const char* what) {
  return fail(TW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
static void resolve(F*& fn, const char* name, bool& ok) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    ok = false;
    return;
  }
  fn = reinterpret_cast<F*>(p);
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    resolve(d.getAttr, "cuDeviceGetAttribute", ok);
    resolve(d.mcCreate, "cuMulticastCreate", ok);
    resolve(d.mcGranularity, "cuMulticastGetGranularity", ok);
    resolve(d.mcAddDevice, "cuMulticastAddDevice", ok);
    resolve(d.mcBindMem, "cuMulticastBindMem", ok);
    resolve(d.mcUnbind, "cuMulticastUnbind", ok);
    resolve(d.memCreate, "cuMemCreate", ok);
    resolve(d.memRelease, "cuMemRelease", ok);
    resolve(d.memGranularity, "cuMemGetAllocationGranularity", ok);
    resolve(d.addrReserve, "cuMemAddressReserve", ok);
    resolve(d.addrFree, "cuMemAddressFree", ok);
    resolve(d.memMap, "cuMemMap", ok);
    resolve(d.memUnmap, "cuMemUnmap", ok);
    resolve(d.memSetAccess, "cuMemSetAccess", ok);
    resolve(d.getErrorString, "cuGetErrorString", ok);
    resolve(d.exportHandle, "cuMemExportToShareableHandle", ok);
    resolve(d.importHandle, "cuMemImportFromShareableHandle", ok);
    d.ok = ok;
  });
  return d;
}

std::string cu_str(CUresult r) {
  const char* s = nullptr;
  if (driver().getErrorString) driver().getErrorString(r, &s);
  return s ? s : ("CUresult " + std::to_string(static_cast<int>(r)));
}

static int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
    cache[device] = n;
  }
  return cache[device];
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---- communicator ------------------------------------------------------------------

static tw_status create_peer(tw_comm* c) {
  c->region = round_up(std::max<size_t>(c->bytes, 1), 256);
  c->total = 3 * c->region + kPadBytes;
  for (int r = 0; r < c->world; ++r) {
    RankBuffers& rb = c->ranks[r];
    cudaError_t e = cudaSetDevice(rb.device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    char* base = nullptr;
    e = cudaMalloc(&base, c->total);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(comm buffers)");
    rb.owns_cuda_malloc = true;
    for (int b = 0; b < 3; ++b) rb.buf[b] = base + b * c->region;
    rb.pad = reinterpret_cast<uint32_t*>(base + 3 * c->region);
    rb.gen = reinterpret_cast<uint32_t*>(base + 3 * c->region + kPadGenOffset);
    rb.err = reinterpret_cast<int*>(base + 3 * c->region + kPadErrOffset);
    e = cudaMemset(base + 3 * c->region, 0, kPadBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(pads)");
  }
  if (!c->colocated) {
    for (int a = 0; a < c->world; ++a) {
      cudaSetDevice(c->ranks[a].device);
      for (int b = 0; b < c->world; ++b) {
        const int da = c->ranks[a].device, db = c->ranks[b].device;
        if (da == db) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, da, db);
        if (!can) return fail(TW_ERR_UNSUPPORTED, "PEER transport: device " + std::to_string(da) +
                                                      " cannot access device " + std::to_string(db));
        cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else if (e != cudaSuccess) {
          return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        }
      }
    }
  }
  return TW_OK;
}

static tw_status create_nvls(tw_comm* c) {
  const Driver& d = driver();
  if (!d.ok) return fail(TW_ERR_UNSUPPORTED, "NVLS: driver multicast entry points unavailable");
  for (const RankBuffers& rb : c->ranks) {
    int mc = 0;
    if (d.getAttr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, rb.device) != CUDA_SUCCESS || !mc)
      return fail(TW_ERR_UNSUPPORTED, "NVLS: device " + std::to_string(rb.device) + " lacks multicast support");
  }
  CUmulticastObjectProp mprop = {};
  mprop.numDevices = static_cast<unsigned>(c->world);
  mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mprop.size = 1;
  size_t mgran = 0;
  CUresult r = d.mcGranularity(&mgran, &mprop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastGetGranularity: " + cu_str(r));
  CUmemAllocationProp aprop = {};
  aprop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  aprop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  aprop.location.id = c->ranks[0].device;
  aprop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  r = d.memGranularity(&agran, &aprop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMemGetAllocationGranularity: " + cu_str(r));
  const size_t gran = std::max(mgran, agran);
  c->region = round_up(std::max<size_t>(c->bytes, 1), gran);
  c->total = 3 * c->region + gran;  // + one granule of signal pads
  mprop.size = c->total;
  r = d.mcCreate(&c->mc, &mprop);
  if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastCreate: " + cu_str(r));
  for (const RankBuffers& rb : c->ranks) {
    r = d.mcAddDevice(c->mc, rb.device);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastAddDevice: " + cu_str(r));
  }
  for (RankBuffers& rb : c->ranks) {
    cudaSetDevice(rb.device);
    aprop.location.id = rb.device;
    r = d.memCreate(&rb.phys, c->total, &aprop, 0);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "cuMemCreate: " + cu_str(r));
    r = d.mcBindMem(c->mc, 0, rb.phys, 0, c->total, 0);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_UNSUPPORTED, "cuMulticastBindMem: " + cu_str(r));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = rb.device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = d.addrReserve(&rb.uc_base, c->total, gran, 0, 0);
    if (r == CUDA_SUCCESS) r = d.memMap(rb.uc_base, c->total, 0, rb.phys, 0);
    if (r == CUDA_SUCCESS) r = d.memSetAccess(rb.uc_base, c->total, &acc, 1);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "unicast map: " + cu_str(r));
    r = d.addrReserve(&rb.mc_base, c->total, gran, 0, 0);
    if (r == CUDA_SUCCESS) r = d.memMap(rb.mc_base, c->total, 0, c->mc, 0);
    if (r == CUDA_SUCCESS) r = d.memSetAccess(rb.mc_base, c->total, &acc, 1);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "multicast map: " + cu_str(r));
    char* uc = reinterpret_cast<char*>(rb.uc_base);
    char* mcp = reinterpret_cast<char*>(rb.mc_base);
    for (int b = 0; b < 3; ++b) {
      rb.buf[b] = uc + b * c->region;
      rb.mc_buf[b] = mcp + b * c->region;
    }
    rb.pad = reinterpret_cast<uint32_t*>(uc + 3 * c->region);
    rb.mc_pad = reinterpret_cast<uint32_t*>(mcp + 3 * c->region);
    rb.gen = reinterpret_cast<uint32_t*>(uc + 3 * c->region + kPadGenOffset);
    rb.err = reinterpret_cast<int*>(uc + 3 * c->region + kPadErrOffset);
    cudaError_t e = cudaMemset(uc + 3 * c->region, 0, kPadBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(pads)");
  }
  for (RankBuffers& rb : c->ranks) {
    cudaSetDevice(rb.device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize(comm create)");
  }
  return TW_OK;
}

void destroy_comm(tw_comm* c) {
  const Driver& d = driver();
  for (RankBuffers& rb : c->ranks) {
    if (rb.ipc_base) {  // a peer's memory imported by this process
      cudaIpcCloseMemHandle(rb.ipc_base);
      continue;
    }
    if (!rb.buf[0] && !rb.phys && !rb.uc_base && !rb.mc_base) continue;  // not owned by this process
    cudaSetDevice(rb.device);
    cudaDeviceSynchronize();
    if (rb.owns_cuda_malloc && rb.buf[0]) cudaFree(rb.buf[0]);
    if (rb.uc_base) {
      d.memUnmap(rb.uc_base, c->total);
      d.addrFree(rb.uc_base, c->total);
    }
    if (rb.mc_base) {
      d.memUnmap(rb.mc_base, c->total);
      d.addrFree(rb.mc_base, c->total);
    }
    if (c->mc && rb.phys) d.mcUnbind(c->mc, rb.device, 0, c->total);
    if (rb.phys) d.memRelease(rb.phys);
  }
  if (c->mc) d.memRelease(c->mc);
  for (cudaEvent_t e : c->join)
    if (e) cudaEventDestroy(e);
  delete c;
}


}  // namespace tw

using namespace tw;

extern "C" {

int tw_abi_version(void) { return TW_ABI_VERSION; }
const char* tw_version(void) { return "tokenweave-b200 0.1 (sm_100a)"; }
const char* tw_last_error(void) { return g_last_error; }

int tw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

tw_status tw_token_shard_map(int64_t num_tokens, int world, int64_t* ranges) {
  clear_error();
  // proj/src/collectives.cpp:26-39
  if (world < 2) return fail(TW_ERR_CONFIG, "token_shard_map: world_size must be >= 2");
  if (num_tokens < 0) return fail(TW_ERR_DIMENSION, "token_shard_map: negative token count");
  if (!ranges) return fail(TW_ERR_DIMENSION, "token_shard_map: null output");
  const int64_t base = num_tokens / world, extra = num_tokens % world;
  int64_t cursor = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t len = base + (r < extra ? 1 : 0);
    ranges[2 * r] = cursor;
    ranges[2 * r + 1] = cursor + len;
    cursor += len;
  }
  return TW_OK;
}

tw_status tw_shard_map_validate(const int64_t* ranges, int world, int64_t total_tokens) {
  clear_error();
  // proj/src/collectives.cpp:14-24
  if (world < 1 || !ranges) return fail(TW_ERR_CONTRACT, "ShardMap: no ranges");
  int64_t cursor = 0;
  for (int r = 0; r < world; ++r) {
    if (ranges[2 * r] != cursor || ranges[2 * r + 1] < ranges[2 * r])
      return fail(TW_ERR_CONTRACT, "ShardMap: ranges must be contiguous, ascending, disjoint");
    cursor = ranges[2 * r + 1];
  }
  if (cursor != total_tokens) return fail(TW_ERR_CONTRACT, "ShardMap: ranges must cover [0, T)");
  return TW_OK;
}

namespace {

// K2 engines (profiles/k2_engines_r01.txt has every A/B behind this policy):
//   Flat  one row per 1024-thread CTA, registers only
//   Rows  the register row engine of tw_rownorm.cuh (also K1's engine)
//   Tma   bulk-copy ring, bulk loads + bulk stores (k2_tma_kernel)
//   Bulk  bulk loads + register stores (k2_bulk_kernel; A/B only)
enum class K2Engine { Flat, Rows, Tma, Bulk };

K2Engine choose_k2_engine(int64_t T, int64_t H, bool bf16, bool vec, int nsm, int sm_budget) {
  static const char* engine_env = std::getenv("TW_K2_ENGINE");
  if (engine_env) {
    if (std::strcmp(engine_env, "rows") == 0) return K2Engine::Rows;
    if (std::strcmp(engine_env, "tma") == 0) return K2Engine::Tma;
    if (std::strcmp(engine_env, "flat") == 0) return K2Engine::Flat;
    return K2Engine::Bulk;
  }
  const int nv = bf16 ? 8 : 4;
  const size_t rbytes = static_cast<size_t>(H) * (bf16 ? 2 : 4);
  // Rows under 12 KB: the register row engine (per-row barrier and bulk-issue
  // costs dominate short rows).  Rows >= 12 KB: the TMA engine (with two
  // consumer row groups it beats the register-store variant at 12 KB rows:
  // H = 6144 bf16, T = 4096: 30.8 vs 41.0 us, tools/k2_groups_ab.py).
  if (!vec || rbytes < 12 * 1024) return K2Engine::Rows;
  // Decode-size batches on the whole GPU (tools/k2_small_graph.py, H = 8192
  // bf16): up to one row per SM the flat engine (no ring to set up; 2.9-3.3 vs
  // 3.7-4.1 us replayed in a CUDA graph, 8.2 vs 8.2-10.2 us cold), up to two
  // rows per SM the row engine (4.1 vs 5.1 us replayed at T = 256).  Under an
  // SM budget the TMA engine moves the most per SM (72 GB/s vs 33 for flat).
  if (sm_budget <= 0) {
    if (T <= nsm && H / nv <= 2048) return K2Engine::Flat;
    if (T <= 2LL * nsm) return K2Engine::Rows;
  }
  return K2Engine::Tma;
}

}  // namespace

tw_status tw_rmsnorm_residual(const void* input, const void* residual, void* residual_out, void* output,
                              const float* weight, int64_t T, int64_t H, float eps, tw_dtype dtype, int sm_budget,
                              void* stream) {
  clear_error();
  // proj/src/numerics.cpp:18-45 (shape, weight, epsilon)
  if (T < 0 || H < 1) return fail(TW_ERR_DIMENSION, "rmsnorm_residual: requires T >= 0 and H >= 1");
  if (!(eps > 0.0f) && eps != 0.0f) return fail(TW_ERR_NUMERIC, "rmsnorm_residual: epsilon must be nonnegative");
  if (dtype != TW_BF16 && dtype != TW_F32) return fail(TW_ERR_CONFIG, "rmsnorm_residual: unknown dtype");
  if (T == 0) return TW_OK;
  if (!input || !residual || !residual_out || !output || !weight)
    return fail(TW_ERR_DIMENSION, "rmsnorm_residual: null buffer");
  const bool bf16 = dtype == TW_BF16;
  const int nv = bf16 ? 8 : 4;
  const bool vec = H % nv == 0 && aligned16(input) && aligned16(residual) && aligned16(residual_out) &&
                   aligned16(output) && aligned16(weight);
  int dev = 0;
  cudaGetDevice(&dev);
  const int nsm = sm_count(dev);
  const int sms = sm_budget > 0 ? std::min(sm_budget, nsm) : nsm;
  const K2Engine engine = choose_k2_engine(T, H, bf16, vec, nsm, sm_budget);
  const bool want_flat = engine == K2Engine::Flat;
  const bool want_rows = engine == K2Engine::Rows;
  const bool tma_store = engine == K2Engine::Tma;
  if (vec && want_flat && H / nv <= 2048) {
    FlatParams f = {};
    f.in = input;
    f.res_in = residual;
    f.res_out = residual_out;
    f.out = output;
    f.weight = weight;
    f.T = T;
    f.H = H;
    f.V = static_cast<int>(H / nv);
    f.eps = eps;
    cudaError_t e = launch_k2_flat(f, bf16, sms, sm_budget > 0, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rmsnorm_residual (flat) launch");
    return TW_OK;
  }
  if (vec && !want_rows) {
    RowPlan bp;
    const uint32_t row_bytes = static_cast<uint32_t>(H * (bf16 ? 2 : 4));
    static const char* cps_env = std::getenv("TW_K2_CTAS_PER_SM");
    // One CTA per SM (an explicit budget really is SMs); concurrency inside
    // the SM comes from two consumer row groups (below).  TW_K2_CTAS_PER_SM
    // keeps the older two-CTA half-ring mode for A/B.
    int cps = 1;
    if (cps_env) cps = std::max(1, std::min(4, std::atoi(cps_env)));
    static const char* ring_env = std::getenv("TW_K2_RING_KB");  // A/B: shared-memory ring budget
    const size_t ring = static_cast<size_t>(ring_env ? std::max(64, std::min(224, std::atoi(ring_env))) : 200) * 1024;
    int stages = static_cast<int>(std::min<size_t>(8, (ring / cps) / (2ull * row_bytes)));
    if (stages < 2 && cps > 1) {  // long rows (>= 25 KB): one CTA per SM keeps a 2+ stage ring
      cps = 1;
      stages = static_cast<int>(std::min<size_t>(8, ring / (2ull * row_bytes)));
    }
    static const char* tpr_env = std::getenv("TW_K2_TPR");  // A/B: consumer threads per row group (overrides)
    const int tpr_pref = tpr_env ? std::max(32, std::min(512, std::atoi(tpr_env))) : (H / nv > 1024 ? 512 : 256);
    if (plan_rows(H, nv, tpr_pref, &bp) && bp.vpt <= 8 && bp.tpr <= kBulkMaxConsumers && stages >= 2) {
      BulkParams q = {};
      q.in = input;
      q.res_in = residual;
      q.res_out = residual_out;
      q.out = output;
      q.weight = weight;
      q.T = T;
      q.H = H;
      q.V = bp.V;
      q.tpr = bp.tpr;
      // Consumer row groups per CTA (k2_tma_kernel), from tools/k2_groups_ab.py:
      // two groups under an SM budget (72 vs 48 GB/s per SM at H = 8192), for
      // short batches (< 48 rows per SM: T = 2048 22.6 vs 28.7 us) and for
      // rows under 16 KB; one group for long batches of >= 16 KB rows (the
      // deeper per-group ring: T = 16384, H = 8192 161.8 vs 172.0 us).
      // TW_K2_GROUPS overrides.
      static const char* groups_env = std::getenv("TW_K2_GROUPS");
      q.groups = (sm_budget > 0 || T < 48LL * nsm || row_bytes < 16 * 1024) ? 2 : 1;
      if (groups_env) q.groups = std::max(1, std::min(2, std::atoi(groups_env)));
      // a group frees its stage one row late, so the ring needs more stages
      // than groups (40 KB rows leave two stages: one group)
      if (q.groups * bp.tpr > kBulkMaxConsumers || stages <= q.groups) q.groups = 1;
      // (512 threads per row for one group measured 1.4 % faster with a clean
      // L2 but 2.5-9 % slower after a producer's dirty lines or back to back:
      // not used, profiles/k2_packed_ab_r02.txt §5; TW_K2_TPR for A/B.)
      q.stages = stages;
      // Loads in flight per SM: with a deep ring (>= 8 stages, rows <= 12.5 KB)
      // two rows ahead of the oldest unarrived one, else the whole ring
      // (tools/k2_policy_check.py A/B, profiles/k2_packed_ab_r02.txt: H = 6144,
      // T = 8192 / 16384 65.5 -> 63.5 / 131 -> 124 us; neutral to +1 us at
      // H = 8192's 6 stages; one row ahead loses 15-20 %).  TW_K2_LOOKAHEAD
      // overrides (0 = the whole ring).
      static const char* la_env = std::getenv("TW_K2_LOOKAHEAD");
      q.lookahead = la_env ? std::max(0, std::atoi(la_env)) : (stages >= 8 ? 2 : 0);
      q.row_bytes = row_bytes;
      q.eps = eps;
      const long long ctas = static_cast<long long>(sms) * cps;
      const int grid = static_cast<int>(std::min<long long>(T, ctas));
      cudaError_t e = launch_k2_bulk(q, bp.vpt, bf16, grid, static_cast<cudaStream_t>(stream), tma_store);
      if (e != cudaSuccess) return cuda_fail(e, "rmsnorm_residual (bulk) launch");
      return TW_OK;
    }
  }
  RowPlan plan;
  // <= 4 vectors per thread: two register sets (the software pipeline) stay spill-free
  if (!plan_rows(H, vec ? nv : 1, H / (vec ? nv : 1) > 1024 ? 512 : 256, &plan))
    return fail(TW_ERR_DIMENSION, "rmsnorm_residual: hidden size too large for the row engine");
  static const char* pipe_env = std::getenv("TW_ROWS_PIPELINE");
  plan.pipeline = pipe_env && pipe_env[0] == '1';
  // An explicit budget is SMs: one CTA each (more CTAs would spread over more SMs).
  const int bpsm = sm_budget > 0 ? 1 : std::max(1, rownorm_blocks_per_sm(plan, bf16, Xport::Local));
  const long long need = (T + plan.groups - 1) / plan.groups;
  const int grid = static_cast<int>(std::min<long long>(need, static_cast<long long>(sms) * bpsm));
  RowParams p = {};
  p.T = T;
  p.H = H;
  p.eps = eps;
  p.in = input;
  p.res_in = residual;
  p.res_out = residual_out;
  p.out = output;
  p.weight = weight;
  cudaError_t e = launch_rownorm(p, plan, bf16, Xport::Local, dim3(grid), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "rmsnorm_residual launch");
  return TW_OK;
}

tw_status tw_count_nonfinite(const void* x, int64_t n, tw_dtype dtype, int* count_dev, void* stream) {
  clear_error();
  if (n < 0) return fail(TW_ERR_DIMENSION, "count_nonfinite: negative size");
  if (n > 0 && (!x || !count_dev)) return fail(TW_ERR_DIMENSION, "count_nonfinite: null buffer");
  cudaError_t e = launch_count_nonfinite(x, n, dtype == TW_BF16, count_dev, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "count_nonfinite launch");
  return TW_OK;
}

tw_status tw_comm_create(int world, const int* devices, size_t buffer_bytes, tw_transport transport, tw_comm_t* out) {
  clear_error();
  if (!out) return fail(TW_ERR_CONFIG, "comm_create: null output");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks)
    return fail(TW_ERR_CONFIG, "comm_create: world must be in [1, " + std::to_string(kMaxRanks) + "]");
  if (!devices) return fail(TW_ERR_CONFIG, "comm_create: null device list");
  if (transport < TW_TRANSPORT_AUTO || transport > TW_TRANSPORT_NVLS_SIM)
    return fail(TW_ERR_CONFIG, "comm_create: unknown transport");
  const int ndev = tw_device_count();
  if (ndev == 0) return fail(TW_ERR_CUDA, "comm_create: no CUDA device visible");
  DeviceGuard guard;
  tw_comm* c = new tw_comm();
  c->world = world;
  c->bytes = buffer_bytes;
  c->ranks.resize(world);
  bool distinct = true;
  c->colocated = true;
  for (int r = 0; r < world; ++r) {
    if (devices[r] < 0 || devices[r] >= ndev) {
      delete c;
      return fail(TW_ERR_CONFIG, "comm_create: device " + std::to_string(devices[r]) + " out of range");
    }
    c->ranks[r].device = devices[r];
    if (devices[r] != devices[0]) c->colocated = false;
    for (int q = 0; q < r; ++q)
      if (devices[q] == devices[r]) distinct = false;
  }
  if (!c->colocated && !distinct) {
    delete c;
    return fail(TW_ERR_CONFIG, "comm_create: ranks must be all on one device or all on distinct devices");
  }
  tw_status st;
  if (transport == TW_TRANSPORT_NVLS_SIM) {
    // test transport: the NVLS kernels on simulated ranks sharing one device
    if (!c->colocated || world < 2) {
      delete c;
      return fail(TW_ERR_UNSUPPORTED, "NVLS_SIM transport needs >= 2 simulated ranks on one device");
    }
    c->transport = TW_TRANSPORT_NVLS_SIM;
    st = create_peer(c);
  } else if (transport == TW_TRANSPORT_NVLS || (transport == TW_TRANSPORT_AUTO && distinct && world >= 2)) {
    c->transport = TW_TRANSPORT_NVLS;
    if (!distinct || world < 2) {
      delete c;
      return fail(TW_ERR_UNSUPPORTED, "NVLS transport needs >= 2 ranks on distinct devices");
    }
    st = create_nvls(c);
    if (st != TW_OK && transport == TW_TRANSPORT_AUTO) {
      // AUTO: fall back to the PEER transport (still the GPU kernel path).
      const std::string why = tw_last_error();
      destroy_comm(c);
      c = new tw_comm();
      c->world = world;
      c->bytes = buffer_bytes;
      c->ranks.resize(world);
      for (int r = 0; r < world; ++r) c->ranks[r].device = devices[r];
      c->transport = TW_TRANSPORT_PEER;
      st = create_peer(c);
    }
  } else {
    c->transport = TW_TRANSPORT_PEER;
    st = create_peer(c);
  }
  if (st != TW_OK) {
    const std::string why = tw_last_error();
    destroy_comm(c);
    return fail(st, why);
  }
  *out = c;
  return TW_OK;
}

tw_status tw_comm_destroy(tw_comm_t comm) {
  clear_error();
  if (!comm) return TW_OK;
  DeviceGuard guard;
  destroy_comm(comm);
  return TW_OK;
}

tw_status tw_comm_info(tw_comm_t comm, int* world, tw_transport* transport, size_t* buffer_bytes) {
  clear_error();
  if (!comm) return fail(TW_ERR_CONFIG, "comm_info: null communicator");
  if (world) *world = comm->world;
  if (transport) *transport = comm->transport;
  if (buffer_bytes) *buffer_bytes = comm->bytes;
  return TW_OK;
}

tw_status tw_comm_local_rank(tw_comm_t comm, int* rank, int* device) {
  clear_error();
  if (!comm) return fail(TW_ERR_CONFIG, "comm_local_rank: null communicator");
  if (rank) *rank = comm->local_rank;
  if (device) *device = comm->ranks[comm->local_rank < 0 ? 0 : comm->local_rank].device;
  return TW_OK;
}

tw_status tw_comm_buffer(tw_comm_t comm, int rank, tw_buffer which, void** device_ptr) {
  clear_error();
  if (!comm || !device_ptr) return fail(TW_ERR_CONFIG, "comm_buffer: null argument");
  if (rank < 0 || rank >= comm->world) return fail(TW_ERR_CONFIG, "comm_buffer: rank out of range");
  if (which < TW_BUF_INPUT || which > TW_BUF_RESIDUAL) return fail(TW_ERR_CONFIG, "comm_buffer: bad buffer id");
  *device_ptr = comm->ranks[rank].buf[which];
  return TW_OK;
}

tw_status tw_comm_multicast_buffer(tw_comm_t comm, int rank, tw_buffer which, void** device_ptr) {
  clear_error();
  if (!comm || !device_ptr) return fail(TW_ERR_CONFIG, "comm_multicast_buffer: null argument");
  if (comm->transport != TW_TRANSPORT_NVLS) return fail(TW_ERR_UNSUPPORTED, "communicator is not NVLS");
  if (rank < 0 || rank >= comm->world) return fail(TW_ERR_CONFIG, "comm_multicast_buffer: rank out of range");
  if (which < TW_BUF_INPUT || which > TW_BUF_RESIDUAL) return fail(TW_ERR_CONFIG, "bad buffer id");
  *device_ptr = comm->ranks[rank].mc_buf[which];
  return TW_OK;
}

tw_status tw_device_alloc(int device, size_t bytes, void** ptr) {
  clear_error();
  if (!ptr) return fail(TW_ERR_CONFIG, "device_alloc: null output");
  *ptr = nullptr;
  DeviceGuard guard;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "device_alloc: cudaSetDevice");
  if (bytes == 0) return TW_OK;
  e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "device_alloc: cudaMalloc");
  return TW_OK;
}

tw_status tw_device_free(int device, void* ptr) {
  clear_error();
  if (!ptr) return TW_OK;
  DeviceGuard guard;
  cudaSetDevice(device);
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) return cuda_fail(e, "device_free");
  return TW_OK;
}

tw_status tw_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
  clear_error();
  if (bytes == 0) return TW_OK;
  if (!dst || !src) return fail(TW_ERR_CONFIG, "memcpy: null pointer");
  cudaError_t e = stream ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream))
                         : cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
  if (e != cudaSuccess) return cuda_fail(e, "memcpy");
  return TW_OK;
}

tw_status tw_device_synchronize(int device) {
  clear_error();
  DeviceGuard guard;
  cudaSetDevice(device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "device_synchronize");
  return TW_OK;
}

tw_status tw_comm_check(tw_comm_t comm) {
  clear_error();
  if (!comm) return fail(TW_ERR_CONFIG, "comm_check: null communicator");
  DeviceGuard guard;
  bool timed_out = false;
  for (const RankBuffers& rb : comm->ranks) {
    cudaSetDevice(rb.device);
    int flag = 0;
    cudaError_t e = cudaMemcpy(&flag, rb.err, sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "comm_check");
    if (flag) {
      timed_out = true;
      cudaMemset(rb.err, 0, sizeof(int));
    }
  }
  if (timed_out) return fail(TW_ERR_TIMEOUT, "cross-rank barrier timed out (a rank was not launched?)");
  return TW_OK;
}

}  // extern "C"

namespace tw {

// Common validation + launch for the fused op (K1) and the AR baseline (K3).
// Single-process communicators launch every rank; a multi-process
// communicator (local_rank >= 0) launches only the rank this process owns.
tw_status comm_launch(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, const int64_t* shard_ranges, void* const* residual_shards,
                      const float* const* weights, float eps, tw_dtype dtype, int sm_budget, unsigned flags,
                      void* const* streams, bool fused) {
  const char* op = fused ? "fused_allreduce_rmsnorm" : "allreduce";
  if (!comm) return fail(TW_ERR_CONFIG, std::string(op) + ": null communicator");
  const int W = comm->world;
  if (W < 2) return fail(TW_ERR_CONFIG, std::string(op) + ": world_size must be >= 2");
  if (T < 0 || H < 1) return fail(TW_ERR_DIMENSION, std::string(op) + ": requires T >= 0 and H >= 1");
  if (dtype != TW_BF16 && dtype != TW_F32) return fail(TW_ERR_CONFIG, std::string(op) + ": unknown dtype");
  const bool bf16 = dtype == TW_BF16;
  const size_t esz = bf16 ? 2 : 4;
  if (token_offset < 0) return fail(TW_ERR_DIMENSION, std::string(op) + ": negative token offset");
  if (static_cast<size_t>(token_offset + T) * static_cast<size_t>(H) * esz > comm->bytes)
    return fail(TW_ERR_DIMENSION, std::string(op) + ": (token_offset+T)*H exceeds the communicator buffer size");
  int64_t local_ranges[2 * kMaxRanks];
  if (!shard_ranges) {
    tw_token_shard_map(T, W, local_ranges);
    shard_ranges = local_ranges;
  }
  tw_status st = tw_shard_map_validate(shard_ranges, W, T);
  if (st != TW_OK) return st;
  auto owned = [&](int r) { return comm->local_rank < 0 || r == comm->local_rank; };
  if (fused) {
    if (!(eps > 0.0f) && eps != 0.0f) return fail(TW_ERR_NUMERIC, "fused_allreduce_rmsnorm: epsilon must be nonnegative");
    if (!weights) return fail(TW_ERR_DIMENSION, "fused_allreduce_rmsnorm: null weight list");
    if (!residual_shards) return fail(TW_ERR_DIMENSION, "fused_allreduce_rmsnorm: null residual list");
    for (int r = 0; r < W; ++r) {
      if (!owned(r)) continue;
      if (!weights[r]) return fail(TW_ERR_DIMENSION, "fused_allreduce_rmsnorm: null weight");
      if (shard_ranges[2 * r + 1] > shard_ranges[2 * r] && !residual_shards[r])
        return fail(TW_ERR_DIMENSION, "fused_allreduce_rmsnorm: null residual shard");
    }
  }
  if (T == 0) return TW_OK;
  const bool sim = comm->transport == TW_TRANSPORT_NVLS_SIM;
  const bool nvls = comm->transport == TW_TRANSPORT_NVLS || sim;  // the NVLS kernels (tw_nvls.cuh)
  const int nv = bf16 ? 8 : 4;
  bool vec = H % nv == 0;
  if (fused) {
    for (int r = 0; r < W && vec; ++r) {
      if (!owned(r)) continue;
      vec = aligned16(weights[r]) && (residual_shards[r] == nullptr || aligned16(residual_shards[r]));
    }
  }
  if (nvls && !vec)
    return fail(TW_ERR_UNSUPPORTED, std::string(op) + ": NVLS transport needs H % " + std::to_string(nv) +
                                        " == 0 and 16-byte aligned buffers");
  RowPlan plan;
  // NVLS: 256-thread row groups (two per CTA), <= 4 vectors per thread so the
  // D + 1 in-flight register sets of the pipeline stay spill-free; PEER holds
  // every rank's vector before summing, so it uses wider groups.
  const long long nvec = H / (vec ? nv : 1);
  if (!plan_rows(H, vec ? nv : 1, nvls ? (nvec > 1024 ? 512 : 256) : 512, &plan))
    return fail(TW_ERR_DIMENSION, std::string(op) + ": hidden size too large for the row engine");
  if (nvls && !nvls_supported(plan))
    return fail(TW_ERR_UNSUPPORTED, std::string(op) + ": NVLS kernel supports H <= " + std::to_string(bf16 ? 16384 : 8192) +
                                        " for this dtype");
  const Xport x = nvls ? Xport::Nvls : Xport::Peer;
  const int depth = nvls_depth_from_flags(flags);

  DeviceGuard guard;
  int budget = sm_budget > 0 ? sm_budget : 8;
  const int dev0 = comm->ranks[comm->local_rank < 0 ? 0 : comm->local_rank].device;
  cudaSetDevice(dev0);
  const int sms = sm_count(dev0);
  // PEER: the bulk-copy pipeline (tw_peer_tma.cuh) whenever the shape fits
  // its ring -- simulated ranks on one B200, T = 8192 x H = 8192: TP = 2
  // 141 vs 182 us, TP = 4 266 vs 279 us (tools/k1_peer_ab.sh).
  // TW_K1_PEER_ENGINE=rows forces the row engine.
  static const char* peer_env = std::getenv("TW_K1_PEER_ENGINE");
  int peer_tma_bpsm = 0;
  if (fused && !nvls && vec && W <= kPeerTmaMaxWorld && !(peer_env && std::strcmp(peer_env, "rows") == 0))
    peer_tma_bpsm = k1_peer_tma_blocks_per_sm(W, static_cast<int>(H / nv), H, bf16);
  if (nvls) {
    // every CTA of every co-launched rank resident for the barrier (the
    // hardware path has one rank per GPU: the budget is simply SMs)
    const int bpsm = fused ? std::max(1, k1_nvls_blocks_per_sm(plan, bf16, sim, depth)) : 1;
    budget = std::min(budget, std::max(1, sms * bpsm / (comm->colocated ? W : 1)));
  } else if (peer_tma_bpsm > 0) {
    const int slots = comm->colocated ? W : 1;
    budget = std::min(budget, std::max(1, sms * peer_tma_bpsm / slots));
  } else if (fused) {
    const int bpsm = std::max(1, rownorm_blocks_per_sm(plan, bf16, x));
    const int slots = comm->colocated ? W : 1;
    // Every CTA of every co-launched rank must be resident for the barrier.
    budget = std::min(budget, std::max(1, sms * bpsm / slots));
  } else {
    budget = std::min(budget, std::max(1, sms / (comm->colocated ? W : 1)));
  }
  budget = std::min(budget, kPadSlots);
  RowParams p = {};
  p.T = T;
  p.H = H;
  p.row_offset = token_offset;
  p.eps = eps;
  // co-located ranks share one GPU: device-scope barrier fences suffice
  // (TW_FORCE_SYS_SCOPE=1 keeps system scope -- measurement of what the
  // fences cost ranks on different GPUs, tools/k1_small.py)
  static const bool force_sys = [] {
    const char* e = std::getenv("TW_FORCE_SYS_SCOPE");
    return e && e[0] == '1';
  }();
  static const bool alias_fence = [] {
    const char* e = std::getenv("TW_NVLS_ALIAS_FENCE");
    return e && e[0] == '1';
  }();
  p.flags = (flags & ~(kDeviceScope | kNvlsDepthMask | kAliasFence)) |
            (comm->colocated && !force_sys ? kDeviceScope : 0u) | (alias_fence ? kAliasFence : 0u);
  p.world = W;
  // Barrier poll bound (~2 s at the default) and the fault-injection hook of
  // the timeout path: TW_FAULT_DROP_ARRIVAL_RANK=r makes rank r never signal,
  // the B200 analogue of the reference's --inject-shard-fault
  // (proj/src/commands.cpp:199-216).  A timed-out communicator is poisoned
  // (its epoch mirror no longer matches the pads): destroy and recreate it.
  const char* spin_env = std::getenv("TW_BARRIER_SPIN_LIMIT");
  const char* drop_env = std::getenv("TW_FAULT_DROP_ARRIVAL_RANK");
  p.spin_limit = spin_env ? std::atoll(spin_env) : (1ll << 25);
  p.drop_arrival_rank = drop_env ? std::atoi(drop_env) : -1;
  for (int q = 0; q < W; ++q) {
    p.peer_in[q] = comm->ranks[q].buf[TW_BUF_INPUT];
    p.peer_out[q] = comm->ranks[q].buf[TW_BUF_OUTPUT];
    p.peer_res[q] = comm->ranks[q].buf[TW_BUF_RESIDUAL];
    p.peer_pad[q] = comm->ranks[q].pad;
  }
  auto fill_slot = [&](RankSlot& s, int r) {
    s.rank = r;
    s.begin = shard_ranges[2 * r];
    s.end = shard_ranges[2 * r + 1];
    s.residual = fused ? residual_shards[r] : nullptr;
    s.weight = fused ? weights[r] : nullptr;
    s.pad = comm->ranks[r].pad;
    s.gen = comm->ranks[r].gen;
  };
  auto launch = [&](const RowParams& pp, dim3 grid, cudaStream_t s) {
    if (nvls)
      return fused ? launch_k1_nvls(pp, plan, bf16, sim, depth, grid, s) : launch_k3_nvls(pp, plan, bf16, sim, grid, s);
    if (peer_tma_bpsm > 0) return launch_k1_peer_tma(pp, W, static_cast<int>(H / nv), bf16, grid, s);
    return fused ? launch_rownorm(pp, plan, bf16, x, grid, s) : launch_allreduce(pp, plan, bf16, x, grid, s);
  };
  if (comm->colocated) {
    p.nslots = W;
    for (int r = 0; r < W; ++r) fill_slot(p.slot[r], r);
    p.err = comm->ranks[0].err;
    cudaStream_t s = streams ? static_cast<cudaStream_t>(streams[0]) : nullptr;
    // one grid for every rank on streams[0]; distinct per-rank streams are
    // joined into it before the launch and released after it, so tw.h's
    // "streams[r] is rank r's stream" ordering holds
    bool distinct = false;
    for (int r = 1; streams && r < W; ++r) distinct |= streams[r] != streams[0];
    if (distinct) {
      if (comm->join.empty()) {
        comm->join.assign(W, nullptr);
        for (int r = 0; r < W; ++r) {
          cudaError_t e = cudaEventCreateWithFlags(&comm->join[r], cudaEventDisableTiming);
          if (e != cudaSuccess) return cuda_fail(e, "comm: join events");
        }
      }
      for (int r = 1; r < W; ++r) {
        if (streams[r] == streams[0]) continue;
        cudaEventRecord(comm->join[r], static_cast<cudaStream_t>(streams[r]));
        cudaStreamWaitEvent(s, comm->join[r], 0);
      }
    }
    cudaError_t e = launch(p, dim3(budget, W), s);
    if (e != cudaSuccess) return cuda_fail(e, op);
    if (distinct) {
      cudaEventRecord(comm->join[0], s);
      for (int r = 1; r < W; ++r)
        if (streams[r] != streams[0]) cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[r]), comm->join[0], 0);
    }
  } else {
    for (int r = 0; r < W; ++r) {
      if (!owned(r)) continue;
      cudaSetDevice(comm->ranks[r].device);
      RowParams pr = p;
      pr.nslots = 1;
      fill_slot(pr.slot[0], r);
      pr.err = comm->ranks[r].err;
      if (nvls) {
        pr.mc_in = comm->ranks[r].mc_buf[TW_BUF_INPUT];
        pr.mc_out = comm->ranks[r].mc_buf[TW_BUF_OUTPUT];
        pr.mc_res = comm->ranks[r].mc_buf[TW_BUF_RESIDUAL];
        pr.mc_pad = comm->ranks[r].mc_pad;
      }
      cudaStream_t s = streams ? static_cast<cudaStream_t>(streams[r]) : nullptr;
      cudaError_t e = launch(pr, dim3(budget, 1), s);
      if (e != cudaSuccess) return cuda_fail(e, op);
    }
  }
  return TW_OK;
}

}  // namespace tw

extern "C" {

tw_status tw_fused_allreduce_rmsnorm_group(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset,
                                           const int64_t* shard_ranges,
                                           void* const* residual_shards, const float* const* weights, float eps,
                                           tw_dtype dtype, int sm_budget, unsigned flags, void* const* streams) {
  clear_error();
  return comm_launch(comm, T, H, token_offset, shard_ranges, residual_shards, weights, eps, dtype, sm_budget, flags,
                     streams, true);
}

tw_status tw_allreduce_group(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, tw_dtype dtype, int sm_budget,
                             void* const* streams) {
  clear_error();
  return comm_launch(comm, T, H, token_offset, nullptr, nullptr, nullptr, 0.0f, dtype, sm_budget, 0u, streams, false);
}

}  // extern "C"
