// Cost of one warp-wide shared-memory atomic add (ATOMS / RED on sm_100a) by
// address pattern: conflict-free, k lanes per bank at distinct addresses, k lanes
// on one address, random, and cross-warp reuse of the same addresses.  One
// 1024-thread CTA per SM, every warp issues `iters` atomics; prints SM clocks per
// warp-instruction (the atomic unit's cost per op).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_pattern atoms_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int RET>
__global__ void __launch_bounds__(1024, 1) k(int pat, int kk, int iters, unsigned long long* clk, uint32_t* sink) {
  extern __shared__ uint32_t sh[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t a;
    const uint32_t base = ((warp * 977u + i * 131u) & 1023u) * 32u;  // per warp/iter region (multiple of 32 words)
    if (pat == 0) a = base + lane;                                   // 32 banks, 32 addresses
    else if (pat == 1) a = base + (lane % (32 / kk)) + (lane / (32 / kk)) * 1024u;  // kk lanes per bank, distinct words
    else if (pat == 2) a = base + (lane % (32 / kk));                // kk lanes per word
    else if (pat == 3) { x = x * 1664525u + 1013904223u; a = x >> 17; }  // random words
    else if (pat == 4) a = lane;                                     // every warp, every iter: same 32 words
    else { x = x * 1664525u + 1013904223u; a = x >> 17; }          // 5: random words, some lanes active
    a &= 32767u;
    const bool on = pat != 5 || ((x >> 3) & 31u) < (uint32_t)kk;   // pat 5: kk of 32 lanes on average
    if (on) {
      if (RET) acc |= atomicAdd(sh + a, 1u);
      else atomicAdd(sh + a, 1u);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = 1;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* clk; uint32_t* sink;
  cudaMalloc(&clk, sms * 8); cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 4096;
  struct P { int pat, kk; const char* name; } ps[] = {
      {0, 1, "conflict-free"}, {1, 2, "2 lanes/bank"}, {1, 4, "4 lanes/bank"}, {1, 8, "8 lanes/bank"},
      {1, 32, "32 lanes/bank"}, {2, 2, "2 lanes/word"}, {2, 4, "4 lanes/word"}, {2, 8, "8 lanes/word"},
      {2, 32, "32 lanes/word"}, {3, 1, "random"}, {4, 1, "same 32 words all warps"},
      {5, 0, "random, 0/32 lanes on"}, {5, 4, "random, ~4/32 lanes on"}, {5, 16, "random, ~16/32 lanes on"}};
  for (auto& p : ps) {
    for (int ret = 0; ret < 2; ++ret) {
      if (ret) k<1><<<sms, 1024, 131072>>>(p.pat, p.kk, iters, clk, sink);
      else k<0><<<sms, 1024, 131072>>>(p.pat, p.kk, iters, clk, sink);
      cudaDeviceSynchronize();
      unsigned long long h[1024]; cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
      double s = 0; for (int i = 0; i < sms; ++i) s += h[i];
      printf("%-26s %s  %.2f clk per warp-op\n", p.name, ret ? "ATOMS(ret)" : "RED      ", s / sms / (32.0 * iters));
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
