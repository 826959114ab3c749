// Probe: device attributes relevant to the NVLS fused collective.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
int main() {
  int n = 0; cudaGetDeviceCount(&n);
  printf("devices=%d\n", n);
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, d);
    int mc = -1, fab = -1, vmm = -1;
    cudaDriverEntryPointQueryResult q;
    PFN_cuDeviceGetAttribute_v2000 getattr = nullptr;
    cudaGetDriverEntryPoint("cuDeviceGetAttribute", (void**)&getattr, cudaEnableDefault, &q);
    getattr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    getattr(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    getattr(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
    printf("dev %d %s sm=%d.%d sms=%d l2=%d smem_optin=%zu multicast=%d fabric=%d vmm=%d\n", d, p.name,
           p.major, p.minor, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, mc, fab, vmm);
  }
  // Try a 1-device multicast object.
  cudaFree(0);
  cudaDriverEntryPointQueryResult q;
  PFN_cuMulticastCreate_v12010 mcCreate = nullptr;
  PFN_cuMulticastGetGranularity_v12010 mcGran = nullptr;
  PFN_cuMulticastAddDevice_v12010 mcAdd = nullptr;
  cudaGetDriverEntryPoint("cuMulticastCreate", (void**)&mcCreate, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastGetGranularity", (void**)&mcGran, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastAddDevice", (void**)&mcAdd, cudaEnableDefault, &q);
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1; prop.size = 2 << 20; prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0; CUresult r = mcGran(&g, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  printf("mc granularity r=%d g=%zu\n", (int)r, g);
  CUmemGenericAllocationHandle h;
  r = mcCreate(&h, &prop);
  printf("mcCreate(1 dev) r=%d\n", (int)r);
  if (r == CUDA_SUCCESS) { r = mcAdd(h, 0); printf("mcAdd r=%d\n", (int)r); }
  return 0;
}
