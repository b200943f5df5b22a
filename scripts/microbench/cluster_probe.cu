// Can a 16-CTA (non-portable) cluster of 1024-thread CTAs with 128 KB of
// dynamic shared memory each be resident on this B200?  Prints the max active
// clusters for sizes 1..16 and times an empty launch.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(int* out) {
  extern __shared__ int sm[];
  cg::cluster_group cl = cg::this_cluster();
  sm[threadIdx.x] = threadIdx.x;
  cl.sync();
  int* peer = cl.map_shared_rank(sm, (cl.block_rank() + 1) % cl.num_blocks());
  if (threadIdx.x == 0) out[blockIdx.x] = peer[5] + (int)cl.num_blocks();
  cl.sync();
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  int* out; cudaMalloc(&out, 64 * sizeof(int));
  for (int c : {1, 2, 4, 8, 12, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, k, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int h[16]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cluster %2d: max active clusters %d (%s), launch %s, %.2f us/launch, out[0]=%d\n", c, nc, cudaGetErrorString(e),
           cudaGetErrorString(e2), ms * 10, h[0]);
  }
  return 0;
}
