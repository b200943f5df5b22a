// cuMulticastCreate straight from the driver API (no Python binding in between).
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  CUdevice d; cuDeviceGet(&d, 0);
  CUcontext c; cuDevicePrimaryCtxRetain(&c, d); cuCtxSetCurrent(c);
  for (int nd = 1; nd <= 2; ++nd) {
    CUmulticastObjectProp p = {};
    p.numDevices = nd; p.size = 2u << 20; p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR; p.flags = 0;
    size_t g = 0;
    CUresult r0 = cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    CUmemGenericAllocationHandle h;
    CUresult r = cuMulticastCreate(&h, &p);
    const char* s = nullptr; cuGetErrorString(r, &s);
    printf("numDevices %d gran %zu (%d) cuMulticastCreate -> %d %s\n", nd, g, (int)r0, (int)r, s ? s : "");
    if (r == CUDA_SUCCESS) {
      CUresult a = cuMulticastAddDevice(h, d);
      printf("  cuMulticastAddDevice -> %d\n", (int)a);
      cuMemRelease(h);
    }
  }
  return 0;
}
