// trie.cu — order-statistic service on the compressed histogram (SURVEY.md §8(f)
// NEXT-3): the dense trie levels, their tapered bit-packed export, and batched
// GetItem / GetIndex queries answered by walking the packed trie.
//
// What it computes:
//  * levels: level p = the leaf histogram; node i of level l counts the keys
//    whose top l bits (MSB-first path, ledger 1) equal i = the sum of its two
//    children (SIBLING SUM).  This is exactly the tree Alg. 1
//     builds key by key; on the GPU only the leaves are
//    counted (hist16.cu) and the internal levels are summed here.  Dense
//    level-ordered layout with computable pointers (Alg. 4):
//    level l at offset 2^l - 1.
//  * pack: per-level tapered width w_l = max(w_min, ceil(log2(capacity+1)) - l)
//    (§III.D.1), promoted by 4 bits while the
//    level's largest counter does not fit (never wrap; ledger 12);
//    counter i of level l at stream bits [off_l + i w_l, off_l + (i+1) w_l),
//    LSB-first in u64 words.
//  * get_item(r): Alg. 2 as order-statistic descent on the
//    LEFT child's count (ledger 4), the key rebuilt from the path (ledger 5);
//    default_value when r >= total.
//  * get_index(v): Alg. 3: the left-subtree counts passed on
//    the way to v = #keys < v (ledger 6).
//
// B200 design: everything here is small and L2-resident (2^(p+1) counters); the
// levels are built by CTAs that each reduce 1,024 leaves in shared memory
// (levels p..p-10), then one CTA finishes the top levels; the pack is a level
// max (warp-reduced atomics), a one-thread plan, and a grid of bit-field ORs;
// queries are one thread each (p dependent L2 reads).
#include "common.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kLeafBlock = 1024;  // leaves per CTA in the first level kernel
constexpr int kLeafLevels = 10;   // levels produced by the first kernel below the leaves

FS_DEVINL uint64_t lvl_off(int l) { return ((uint64_t)1 << l) - 1; }

// Levels p .. max(p - 10, 0) from 1,024-leaf blocks.
__global__ void __launch_bounds__(512) k_levels_low(const uint64_t* __restrict__ leaves, int p,
                                                    uint64_t* __restrict__ levels) {
  __shared__ uint64_t sh[kLeafBlock];
  const uint32_t tid = threadIdx.x;
  const uint64_t nleaf = (uint64_t)1 << p;
  const uint64_t base = (uint64_t)blockIdx.x * kLeafBlock;
  const uint32_t cnt = (uint32_t)min((uint64_t)kLeafBlock, nleaf - base);
  for (uint32_t i = tid; i < cnt; i += blockDim.x) {
    const uint64_t x = leaves[base + i];
    sh[i] = x;
    levels[lvl_off(p) + base + i] = x;
  }
  __syncthreads();
  uint32_t width = cnt;
  for (int l = p - 1; l >= 0 && l >= p - kLeafLevels; --l) {
    width >>= 1;
    uint64_t v[2] = {0, 0};
    for (uint32_t i = tid, k = 0; i < width; i += blockDim.x, ++k) v[k] = sh[2 * i] + sh[2 * i + 1];
    __syncthreads();
    for (uint32_t i = tid, k = 0; i < width; i += blockDim.x, ++k) {
      sh[i] = v[k];
      levels[lvl_off(l) + (base >> (p - l)) + i] = v[k];
    }
    __syncthreads();
  }
}

// Levels below p - 10 (p > 10): one CTA, level by level from global memory.
__global__ void __launch_bounds__(1024) k_levels_top(int p, uint64_t* __restrict__ levels) {
  for (int l = p - kLeafLevels - 1; l >= 0; --l) {
    for (uint64_t i = threadIdx.x; i < ((uint64_t)1 << l); i += blockDim.x)
      levels[lvl_off(l) + i] = levels[lvl_off(l + 1) + 2 * i] + levels[lvl_off(l + 1) + 2 * i + 1];
    __syncthreads();
  }
}

// Largest counter of every level (mx zeroed by the caller): blockIdx.y = level,
// each CTA reduces a 4,096-node chunk and issues one atomic.
constexpr int kMaxChunk = 4096;
__global__ void __launch_bounds__(256) k_level_max(const uint64_t* __restrict__ levels,
                                                   unsigned long long* __restrict__ mx) {
  __shared__ unsigned long long wmax[8];
  const int l = blockIdx.y;
  const uint64_t nodes = (uint64_t)1 << l;
  const uint64_t c0 = (uint64_t)blockIdx.x * kMaxChunk;
  if (c0 >= nodes) return;
  const uint64_t c1 = min(c0 + kMaxChunk, nodes);
  unsigned long long m = 0;
  for (uint64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) m = max(m, (unsigned long long)levels[lvl_off(l) + i]);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(kFull, m, d));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = max(m, wmax[w]);
    if (m) atomicMax(&mx[l], m);
  }
}

// Widths and bit offsets (one thread).  widths[0] = -1 when the stream does not fit.
__global__ void k_pack_plan(const unsigned long long* __restrict__ mx, int p, uint64_t capacity, int min_width,
                            uint64_t words, int32_t* __restrict__ widths, uint64_t* __restrict__ off) {
  if (threadIdx.x || blockIdx.x) return;
  int full = 0;
  while (full < 64 && ((full == 64 ? ~0ull : ((1ull << full) - 1)) < capacity)) ++full;  // ceil(log2(capacity+1))
  uint64_t o = 0;
  for (int l = 0; l <= p; ++l) {
    int w = full - l;
    if (w < min_width) w = min_width;
    while (w < 64 && (mx[l] >> w) != 0) w += 4;
    if (w > 64) w = 64;
    widths[l] = w;
    off[l] = o;
    o += ((uint64_t)1 << l) * (uint64_t)w;
  }
  off[p + 1] = o;
  if ((o + 63) / 64 > words) widths[0] = -1;
}

__global__ void __launch_bounds__(256) k_pack(const uint64_t* __restrict__ levels, int p,
                                              const int32_t* __restrict__ widths, const uint64_t* __restrict__ off,
                                              unsigned long long* __restrict__ packed) {
  if (widths[0] < 0) return;
  const uint64_t total = ((uint64_t)2 << p) - 1;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const int l = 63 - __clzll((long long)(g + 1));
    const uint64_t i = g - lvl_off(l);
    const int w = widths[l];
    const uint64_t x = levels[g];
    if (!x) continue;  // the stream is zeroed
    const uint64_t pos = off[l] + i * (uint64_t)w;
    const uint32_t sh = (uint32_t)(pos & 63);
    atomicOr(&packed[pos >> 6], (unsigned long long)(x << sh));
    if (sh + w > 64) atomicOr(&packed[(pos >> 6) + 1], (unsigned long long)(x >> (64 - sh)));
  }
}

struct PackedTrie {
  const int32_t* widths;
  const uint64_t* off;
  const uint64_t* packed;
  FS_DEVINL uint64_t count(int l, uint64_t i) const {
    const int w = __ldg(widths + l);
    const uint64_t pos = __ldg(off + l) + i * (uint64_t)w;
    const uint32_t sh = (uint32_t)(pos & 63);
    uint64_t x = __ldg(packed + (pos >> 6)) >> sh;
    if (sh + w > 64) x |= __ldg(packed + (pos >> 6) + 1) << (64 - sh);
    return w >= 64 ? x : (x & ((1ull << w) - 1));
  }
};

__global__ void __launch_bounds__(256) k_get_item(PackedTrie t, int p, const uint64_t* __restrict__ ranks, uint64_t q,
                                                  uint64_t default_value, uint64_t* __restrict__ items) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < q; k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = ranks[k];
    if (r >= t.count(0, 0)) {
      items[k] = default_value;
      continue;
    }
    uint64_t node = 0;
    for (int l = 0; l < p; ++l) {
      const uint64_t left = node << 1;
      const uint64_t cl = t.count(l + 1, left);
      if (r < cl) {
        node = left;
      } else {
        r -= cl;
        node = left | 1u;
      }
    }
    items[k] = node;
  }
}

__global__ void __launch_bounds__(256) k_get_index(PackedTrie t, int p, const uint64_t* __restrict__ values,
                                                   uint64_t q, uint64_t* __restrict__ indices) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < q; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = values[k];
    uint64_t idx = 0, node = 0;
    for (int l = 0; l < p; ++l) {
      const uint64_t bit = (v >> (p - 1 - l)) & 1u;
      const uint64_t left = node << 1;
      if (bit) idx += t.count(l + 1, left);
      node = left | bit;
    }
    indices[k] = idx;
  }
}

__global__ void __launch_bounds__(256) k_hist_merge(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                                    uint64_t* __restrict__ out, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

unsigned grid_for(uint64_t work, unsigned threads) {
  const uint64_t cap = (uint64_t)device_info().sm_count * 8;
  uint64_t g = (work + threads - 1) / threads;
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

}  // namespace

cudaError_t launch_trie_levels(const uint64_t* leaves, int p, uint64_t* levels, cudaStream_t s) {
  const uint64_t nleaf = (uint64_t)1 << p;
  k_levels_low<<<(unsigned)((nleaf + kLeafBlock - 1) / kLeafBlock), 512, 0, s>>>(leaves, p, levels);
  if (p > kLeafLevels) k_levels_top<<<1, 1024, 0, s>>>(p, levels);
  return cudaGetLastError();
}

cudaError_t launch_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int32_t* widths,
                             uint64_t* off, uint64_t* packed, uint64_t words, unsigned long long* mx,
                             cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * (p + 1), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(packed, 0, sizeof(uint64_t) * words, s)) != cudaSuccess) return e;
  const uint64_t total = ((uint64_t)2 << p) - 1;
  const uint64_t chunks = (((uint64_t)1 << p) + kMaxChunk - 1) / kMaxChunk;
  k_level_max<<<dim3((unsigned)chunks, (unsigned)(p + 1)), 256, 0, s>>>(levels, mx);
  k_pack_plan<<<1, 32, 0, s>>>(mx, p, capacity, min_width, words, widths, off);
  k_pack<<<grid_for(total, 256), 256, 0, s>>>(levels, p, widths, off, (unsigned long long*)packed);
  return cudaGetLastError();
}

cudaError_t launch_get_item(const int32_t* widths, const uint64_t* off, const uint64_t* packed, int p,
                            const uint64_t* ranks, uint64_t q, uint64_t default_value, uint64_t* items,
                            cudaStream_t s) {
  k_get_item<<<grid_for(q, 256), 256, 0, s>>>(PackedTrie{widths, off, packed}, p, ranks, q, default_value, items);
  return cudaGetLastError();
}

cudaError_t launch_get_index(const int32_t* widths, const uint64_t* off, const uint64_t* packed, int p,
                             const uint64_t* values, uint64_t q, uint64_t* indices, cudaStream_t s) {
  k_get_index<<<grid_for(q, 256), 256, 0, s>>>(PackedTrie{widths, off, packed}, p, values, q, indices);
  return cudaGetLastError();
}

cudaError_t launch_hist_merge(const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t count, cudaStream_t s) {
  k_hist_merge<<<grid_for(count, 256), 256, 0, s>>>(a, b, out, count);
  return cudaGetLastError();
}

}  // namespace fs
