// Throughput of the two counting units a histogram can use on sm_100a:
// shared-memory atomics (ATOMS, packed u16 halves as in k_hist16) and L2
// reductions (RED.E.ADD to a 65,536-word global table), alone and mixed in
// one warp, on random (LCG) bins.  Prints G-increments/s for each variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>  // 0: smem only, 1: global red only, 2: mix (1 of R to global), 3: smem, returns OR-ed
__global__ void __launch_bounds__(1024) k(uint32_t* g, int iters, int R) {
  extern __shared__ uint32_t sh[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t v = x >> 16;
    if (MODE == 3) {
      acc |= atomicAdd(sh + (v >> 1), 1u << ((v & 1) * 16));
    } else if (MODE == 0 || (MODE == 2 && (i % R) != 0)) {
      atomicAdd(sh + (v >> 1), 1u << ((v & 1) * 16));
    } else {
      asm volatile("red.global.add.u32 [%0], 1;" ::"l"(g + v) : "memory");
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32768; i += blockDim.x)
    if (sh[i] == 0xFFFFFFFFu || acc == 0x12345678u) g[i] = 1;  // keep the smem work alive
}

// The histogram's core loop alone: 16 keys (two 16-B vectors) per thread per
// group, grid-strided, next group loaded before the current group's atomics,
// returns OR-ed (as k_hist16 uses them for overflow detection).
template <bool RET>
__global__ void __launch_bounds__(1024) kh(const uint4* __restrict__ in, uint64_t nvec, uint32_t* g) {
  extern __shared__ uint32_t sh[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 2;
  uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  uint4 c0 = i < nvec ? __ldcs(in + i) : make_uint4(0, 0, 0, 0), c1 = i + 1 < nvec ? __ldcs(in + i + 1) : make_uint4(0, 0, 0, 0);
  for (; i < nvec; i += stride) {
    const uint64_t j = i + stride;
    uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
    if (j < nvec) { n0 = __ldcs(in + j); n1 = __ldcs(in + j + 1); }
    const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t lo = w[t] & 0xFFFFu, hi = w[t] >> 16;
      if (RET) {
        acc |= atomicAdd(sh + (lo >> 1), 1u << ((lo & 1) * 16));
        acc |= atomicAdd(sh + (hi >> 1), 1u << ((hi & 1) * 16));
      } else {
        atomicAdd(sh + (lo >> 1), 1u << ((lo & 1) * 16));
        atomicAdd(sh + (hi >> 1), 1u << ((hi & 1) * 16));
      }
    }
    c0 = n0; c1 = n1;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 32768; t += blockDim.x)
    if (sh[t] == 0xFFFFFFFFu || acc == 0x12345678u) g[t] = 1;
}

__global__ void fill(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32;
    p[i] = (uint32_t)z;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* g;
  cudaMalloc(&g, 65536 * 4);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int R) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      kern<<<sms, 1024, 131072>>>(g, iters, R);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%-24s R=%2d  %.3f ms  %.1f G inc/s\n", name, R, ms, (double)sms * 1024 * iters / (ms * 1e6));
    }
  };
  run("smem", k<0>, 1);
  run("smem, returns used", k<3>, 1);
  run("global red", k<1>, 1);
  for (int R : {2, 3, 4, 6, 8, 16}) run("mix (1/R global)", k<2>, R);
  {
    const uint64_t nkeys = 1ull << 28;
    uint4* in;
    cudaMalloc(&in, nkeys * 2);
    fill<<<1184, 256>>>((uint32_t*)in, nkeys / 2);
    cudaFuncSetAttribute(kh<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncSetAttribute(kh<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int ret = 0; ret < 2; ++ret)
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        if (ret) kh<true><<<sms, 1024, 131072>>>(in, nkeys / 8, g);
        else kh<false><<<sms, 1024, 131072>>>(in, nkeys / 8, g);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 3) printf("hist core 2^28 keys ret=%d  %.1f us  %.1f GB/s\n", ret, ms * 1e3, nkeys * 2 / (ms * 1e6));
      }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
