// hist16.cu — stage 1 of the u16 path: the per-SM compressed histogram (G1).
//
// What it computes (§III.B.1 Fractal RMW, Alg. 1):
// every key increments the counter of the leaf its MSB-first bit path selects;
// at p = 16 the leaf slot is the key itself (ledger 1; computable pointers,
// PAPER.md:196-215).  The trie's internal levels are sums of leaves (SIBLING
// SUM), so only the leaf level is materialised; the scan builds
// the rest implicitly.
//
// B200 design:
//  * One CTA of 1024 threads per SM; the 65,536-bin local tree lives in shared
//    memory as 16-bit counters packed two per 32-bit word (128 KB): counter-width
//    tapering (§III.D.1) is what makes a privatised 65,536-bin
//    histogram fit in one SM (n_L = W/w_c = 2 counters per word).
//    Bin v lives in word v>>1, half v&1, so the packed partial is exactly a u16
//    array indexed by bin.
//  * Keys stream in as 128-bit loads (8 keys) with evict-first, one vector
//    look-ahead per unrolled group to keep bytes in flight.
//  * Overflow ("Counter Width Compression and Overflow", ledger 12):
//    never wraps.  Every shared atomic returns the old word; a thread that sees
//    either half >= THETA (2^14) atomically exchanges the word with 0 and adds
//    both halves to the global u64 spill array.  Between the increment that
//    lifts a counter to >= THETA and the first exchange, each thread can add at
//    most the keys of one unrolled group (UNROLL*8) to it, because it checks the
//    returned values before its next group; so a counter never exceeds
//    THETA + 255 + 1024*UNROLL*8 = 49,407 < 65,536 (UNROLL = 4).  No barrier.
//  * Runs of equal keys (sorted or constant inputs, ledger 21-22) are aggregated:
//    a thread whose 8 keys are equal issues one +8; a warp whose 256 keys are
//    all equal issues one +256 from lane 0 (same-address atomics serialise).
//  * At the end the CTA writes its 128 KB partial to partials[blockIdx.x]
//    (L2-resident) for the merge in scan.cu (PAPER.md:89 two-step merge).
#include "common.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 1024;
constexpr int kUnroll = 4;              // 128-bit vectors per thread per group
constexpr uint32_t kHotMask = 0xC000C000u;  // either 16-bit half >= 2^14

static_assert(16384 + 255 + kThreads * kUnroll * 8 < 65536, "spill bound violated");

FS_DEVINL void spill_word(uint32_t* sh, uint32_t w, unsigned long long* spill) {
  const uint32_t x = atomicExch(&sh[w], 0u);
  if (x & 0xFFFFu) atomicAdd(&spill[2 * w], (unsigned long long)(x & 0xFFFFu));
  if (x >> 16) atomicAdd(&spill[2 * w + 1], (unsigned long long)(x >> 16));
}

// Add `cnt` (<= 256) to bin k; spill if the counter word was hot.
FS_DEVINL void add_key(uint32_t* sh, uint32_t k, uint32_t cnt, unsigned long long* spill) {
  const uint32_t w = k >> 1;
  const uint32_t old = atomicAdd(&sh[w], (k & 1u) ? (cnt << 16) : cnt);
  if (old & kHotMask) spill_word(sh, w, spill);
}

// Plain path: 8 independent atomics, returns checked after all are issued.
FS_DEVINL void add8(uint32_t* sh, const uint4& v, unsigned long long* spill) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t old[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t lo = w[j] & 0xFFFFu, hi = w[j] >> 16;
    old[2 * j] = atomicAdd(&sh[lo >> 1], (lo & 1u) ? 0x10000u : 1u);
    old[2 * j + 1] = atomicAdd(&sh[hi >> 1], (hi & 1u) ? 0x10000u : 1u);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (old[2 * j] & kHotMask) spill_word(sh, (w[j] & 0xFFFFu) >> 1, spill);
    if (old[2 * j + 1] & kHotMask) spill_word(sh, w[j] >> 17, spill);
  }
}

FS_DEVINL bool all8_equal(const uint4& v) {
  return (v.x == v.y) & (v.y == v.z) & (v.z == v.w) & ((v.x >> 16) == (v.x & 0xFFFFu));
}

// Aggregating path for a vector when the warp has runs of equal keys.
FS_DEVINL void add8_agg(uint32_t* sh, const uint4& v, unsigned long long* spill) {
  const bool eq = all8_equal(v);
  const uint32_t k0 = v.x & 0xFFFFu;
  const uint32_t lane0_key = __shfl_sync(kFull, k0, 0);  // every lane must execute the shuffle
  const bool warp_same = __all_sync(kFull, eq && k0 == lane0_key);
  if (warp_same) {
    if (lane_id() == 0) add_key(sh, k0, 256u, spill);
  } else if (eq) {
    add_key(sh, k0, 8u, spill);
  } else {
    add8(sh, v, spill);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_hist16(const uint16_t* __restrict__ keys, uint64_t n, uint64_t head, uint64_t nvec,
             uint32_t* __restrict__ partials, unsigned long long* __restrict__ spill) {
  extern __shared__ uint4 smem_v4[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem_v4);

  // zero the local tree (128 KB)
#pragma unroll
  for (int i = 0; i < kHistWords / 4 / kThreads; ++i) smem_v4[threadIdx.x + i * kThreads] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  // Unaligned head and ragged tail (< 8 + 7 keys) go to the last CTA, one key per thread.
  if (blockIdx.x == gridDim.x - 1) {
    const uint64_t tail0 = head + nvec * 8;
    const uint64_t nscalar = head + (n - tail0);
    for (uint64_t t = threadIdx.x; t < nscalar; t += kThreads) {
      const uint64_t idx = t < head ? t : tail0 + (t - head);
      add_key(sh, keys[idx], 1u, spill);
    }
  }

  const uint4* __restrict__ vec = reinterpret_cast<const uint4*>(keys + head);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;

  // Main loop: groups of kUnroll vectors at grid stride.  The bound is tested on
  // the warp's last lane so the whole warp iterates together (warp collectives).
  const uint64_t warp_tail = 31 - lane_id();
  for (; i + warp_tail + (kUnroll - 1) * stride < nvec; i += kUnroll * stride) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream_v4(vec + i + u * stride);
    bool runs = false;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) runs |= all8_equal(v[u]);
    if (__any_sync(kFull, runs)) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) add8_agg(sh, v[u], spill);
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) add8(sh, v[u], spill);
    }
  }
  // Remainder vectors (fewer than kUnroll per thread).
  for (; i < nvec; i += stride) add8(sh, ld_stream_v4(vec + i), spill);

  __syncthreads();
  // Flush the local tree: the first step of the two-step merge.
  uint4* dst = reinterpret_cast<uint4*>(partials + (uint64_t)blockIdx.x * kHistWords);
#pragma unroll
  for (int j = 0; j < kHistWords / 4 / kThreads; ++j) dst[threadIdx.x + j * kThreads] = smem_v4[threadIdx.x + j * kThreads];
}

}  // namespace

int hist16_grid(uint64_t n) {
  const uint64_t want = (n + 65535) / 65536;  // keep >= 64K keys per CTA: the flush is 128 KB
  const uint64_t sms = (uint64_t)device_info().sm_count;
  uint64_t g = want < sms ? want : sms;
  return g ? (int)g : 1;
}

cudaError_t launch_hist16(const uint16_t* keys, uint64_t n, uint32_t* partials, unsigned long long* spill, int grid,
                          cudaStream_t s) {
  static_assert(kHistWords % (4 * kThreads) == 0, "flush mapping");
  constexpr int smem = kHistWords * 4;
  cudaError_t e = cudaFuncSetAttribute(k_hist16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // 16-byte aligned body: head keys before it, nvec full vectors, then the tail.
  const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
  uint64_t head = ((16 - (addr & 15)) & 15) / 2;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 8;
  k_hist16<<<grid, kThreads, smem, s>>>(keys, n, head, nvec, partials, spill);
  return cudaGetLastError();
}

}  // namespace fs
