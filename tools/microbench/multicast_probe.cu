// NVLS multicast probe: can this box create a multicast object (for a multimem.st
// fused exchange)?  nvcc -gencode arch=compute_100a,code=sm_100a multicast_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  CUdevice d; cuDeviceGet(&d, 0);
  CUcontext ctx; cuCtxCreate(&ctx, 0, d);
  unsigned long long types[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int t = 0; t < 3; ++t) {
    CUmulticastObjectProp p = {};
    p.numDevices = 1; p.size = 2 << 20; p.handleTypes = types[t];
    CUmemGenericAllocationHandle h;
    CUresult r = cuMulticastCreate(&h, &p);
    const char* s = nullptr; cuGetErrorString(r, &s);
    printf("handleTypes=%llu cuMulticastCreate rc=%d (%s)\n", types[t], (int)r, s ? s : "?");
    if (r == CUDA_SUCCESS) {
      r = cuMulticastAddDevice(h, d);
      cuGetErrorString(r, &s);
      printf("  addDevice rc=%d (%s)\n", (int)r, s);
      CUmemAllocationProp ap = {};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
      ap.requestedHandleTypes = (CUmemAllocationHandleType)types[t];
      CUmemGenericAllocationHandle mem;
      r = cuMemCreate(&mem, 2 << 20, &ap, 0); cuGetErrorString(r, &s); printf("  memCreate rc=%d (%s)\n", (int)r, s);
      r = cuMulticastBindMem(h, 0, mem, 0, 2 << 20, 0); cuGetErrorString(r, &s); printf("  bindMem rc=%d (%s)\n", (int)r, s);
      CUdeviceptr va; r = cuMemAddressReserve(&va, 2 << 20, 2 << 20, 0, 0);
      r = cuMemMap(va, 2 << 20, 0, h, 0); cuGetErrorString(r, &s); printf("  map mc rc=%d (%s)\n", (int)r, s);
    }
  }
  return 0;
}
