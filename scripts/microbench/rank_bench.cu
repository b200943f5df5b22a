// Throughput of warp-level "peers" computation on sm_100a: 8-ballot multisplit
// (compiler form and inline-PTX form) vs __match_any_sync, 2^24 items per warp-slot.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t peers_ballot(uint32_t d) {
  uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t v = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? v : ~v;
  }
  return peers;
}
__device__ __forceinline__ uint32_t peers_ptx(uint32_t d) {
  uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 v, m;\n\t"
        "and.b32 m, %1, %2;\n\tsetp.ne.u32 p, m, 0;\n\t"
        "vote.sync.ballot.b32 v, p, 0xffffffff;\n\t"
        "selp.b32 m, 0, -1, p;\n\t"
        "lop3.b32 %0, %0, v, m, 0x60;\n\t}"   // peers & (v ^ m): m = ~0 when bit is 0 -> ~v
        : "+r"(peers) : "r"(d), "r"(1u << b));
  }
  return peers;
}
__device__ __forceinline__ uint32_t peers_match(uint32_t d) { return __match_any_sync(0xFFFFFFFFu, d); }

template <int V>
__global__ void k(uint32_t* out, int iters) {
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t d = x >> 24;
    uint32_t p = V == 0 ? peers_ballot(d) : V == 1 ? peers_ptx(d) : peers_match(d);
    acc += __popc(p & ((1u << (threadIdx.x & 31)) - 1));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  const int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* nm[3] = {"ballot (C++)", "ballot (PTX)", "match.any"};
  for (int rep = 0; rep < 2; ++rep)
  for (int v = 0; v < 3; ++v) {
    cudaEventRecord(a);
    if (v == 0) k<0><<<148 * 2, 1024>>>(out, iters);
    if (v == 1) k<1><<<148 * 2, 1024>>>(out, iters);
    if (v == 2) k<2><<<148 * 2, 1024>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double warp_ops = 148.0 * 2 * 32 * iters;
    printf("%-14s %8.3f ms  %6.2f cycles per warp-op per SM (1.9 GHz)\n", nm[v], ms, ms * 1e-3 * 1.9e9 / (warp_ops / 148));
  }
  uint32_t* p1; uint32_t* p2; // correctness: compare ballot forms vs match
  return 0;
}
