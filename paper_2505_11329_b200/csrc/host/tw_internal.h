// tw_internal.h -- host-side internals of libtw.so (communicator, errors).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tw/tw.h"

namespace tw {

// Thread-local last-error message behind tw_last_error().
void set_error(const std::string& msg);
void clear_error();
tw_status fail(tw_status code, const std::string& msg);
tw_status cuda_fail(cudaError_t e, const char* what);

// Driver API entry points resolved through cudaGetDriverEntryPoint, so the
// library has no link-time dependency on libcuda (it loads on GPU-less hosts).
struct Driver {
  bool ok = false;
  CUresult (*getAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) =
      nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*memGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  CUresult (*exportHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) =
      nullptr;
  CUresult (*importHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
};
const Driver& driver();

struct RankBuffers {
  int device = 0;
  void* buf[3] = {nullptr, nullptr, nullptr};  // INPUT, OUTPUT, RESIDUAL (unicast)
  uint32_t* pad = nullptr;                      // signal counters (unicast)
  uint32_t* gen = nullptr;                      // per-CTA-index launch generations
  int* err = nullptr;                           // barrier-timeout flag
  // NVLS
  void* mc_buf[3] = {nullptr, nullptr, nullptr};
  uint32_t* mc_pad = nullptr;
  CUmemGenericAllocationHandle phys = 0;
  CUdeviceptr uc_base = 0, mc_base = 0;
  bool owns_cuda_malloc = false;
  void* ipc_base = nullptr;  // multi-process PEER: a peer's allocation opened via cudaIpcOpenMemHandle
};

}  // namespace tw

struct tw_comm {
  int world = 0;
  tw_transport transport = TW_TRANSPORT_PEER;
  size_t bytes = 0;         // per symmetric buffer
  size_t region = 0;        // aligned per-buffer stride inside one allocation
  size_t total = 0;         // bytes of one rank's allocation
  bool colocated = false;   // every rank on the same device
  std::vector<tw::RankBuffers> ranks;
  CUmemGenericAllocationHandle mc = 0;
  int local_rank = -1;      // >= 0: multi-process communicator owning only this rank
  // co-located launches go on streams[0]: these join the other ranks' streams
  // before (rank r's event) and after (slot 0) the launch
  std::vector<cudaEvent_t> join;
};

namespace tw {
tw_status comm_launch(tw_comm_t comm, int64_t T, int64_t H, int64_t token_offset, const int64_t* shard_ranges,
                      void* const* residual_shards, const float* const* weights, float eps, tw_dtype dtype,
                      int sm_budget, unsigned flags, void* const* streams, bool fused);
size_t round_up(size_t x, size_t a);
std::string cu_str(CUresult r);
void destroy_comm(tw_comm* c);
}  // namespace tw
