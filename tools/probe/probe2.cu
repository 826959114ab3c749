// Probe: which cuMulticastCreate configurations a 1-GPU B200 box accepts.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
int main() {
  cudaFree(0);
  cudaDriverEntryPointQueryResult q;
  PFN_cuMulticastCreate_v12010 mcCreate = nullptr;
  PFN_cuMulticastGetGranularity_v12010 mcGran = nullptr;
  PFN_cuMulticastAddDevice_v12010 mcAdd = nullptr;
  PFN_cuGetErrorString_v6000 errstr = nullptr;
  cudaGetDriverEntryPoint("cuMulticastCreate", (void**)&mcCreate, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastGetGranularity", (void**)&mcGran, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastAddDevice", (void**)&mcAdd, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuGetErrorString", (void**)&errstr, cudaEnableDefault, &q);
  unsigned long long types[] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR | CU_MEM_HANDLE_TYPE_FABRIC};
  for (unsigned nd : {1u, 2u}) {
    for (auto t : types) {
      CUmulticastObjectProp prop = {};
      prop.numDevices = nd;
      prop.handleTypes = t;
      prop.size = 1;
      size_t g = 0;
      CUresult r = mcGran(&g, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
      prop.size = g ? g * 4 : (8 << 20);
      CUmemGenericAllocationHandle h = 0;
      CUresult rc = mcCreate(&h, &prop);
      const char* s = nullptr;
      errstr(rc, &s);
      CUresult ra = CUDA_ERROR_UNKNOWN;
      if (rc == CUDA_SUCCESS) ra = mcAdd(h, 0);
      const char* s2 = nullptr;
      errstr(ra, &s2);
      printf("numDevices=%u handleTypes=%llu gran_rc=%d gran=%zu create=%d (%s) add=%d (%s)\n", nd, t, (int)r, g,
             (int)rc, s ? s : "?", (int)ra, rc == CUDA_SUCCESS ? (s2 ? s2 : "?") : "-");
    }
  }
  return 0;
}
