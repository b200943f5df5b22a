// Phase timing of the one-cluster u16 sort (small16.cu built with -DFS_SMALL_TRACE).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFS_SMALL_TRACE -I../../include
//        -I../../paper_2605_10390_b200/csrc -o small_trace small_trace.cu
#include <cstdio>
#include <cstdlib>
#include "../../paper_2605_10390_b200/csrc/small16.cu"
__global__ void gen(uint16_t* k, uint64_t n, int mode) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
    k[i] = mode ? 0xA5A5 : (uint16_t)z;
  }
}
int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1 << 20);
  int mode = argc > 2 ? atoi(argv[2]) : 0;
  uint16_t *k, *o; unsigned long long* sp; uint32_t* part;
  cudaMalloc(&k, n * 2); cudaMalloc(&o, n * 2); cudaMalloc(&sp, 65536 * 8); cudaMalloc(&part, 16 * 131072);
  gen<<<592, 256>>>(k, n, mode); cudaDeviceSynchronize();
  for (int rep = 0; rep < 5; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = fs::launch_sort16_small(k, n, o, sp, part, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long tr[16][16]; cudaMemcpyFromSymbol(tr, g_small_trace, sizeof(tr));
    printf("rep %d (%s) event %.1f us |", rep, cudaGetErrorString(e), ms * 1e3);
    for (int i = 1; i < 7; ++i) printf(" p%d %.2f", i, (tr[0][i] - tr[0][i - 1]) / 1e3);
    printf(" | merge-loads %.2f scan %.2f | base %.2f chunks %.2f edges %.2f", (tr[0][9] - tr[0][2]) / 1e3,
           (tr[0][3] - tr[0][9]) / 1e3, (tr[0][7] - tr[0][4]) / 1e3, (tr[0][8] - tr[0][7]) / 1e3,
           (tr[0][5] - tr[0][8]) / 1e3);
    printf("\n");
  }
  return 0;
}
