// small16.cu — the whole u16 keys-only sort (rows a1–a5) in ONE launch for
// small inputs (n <= small16_max_n()): one thread-block cluster of 16 CTAs
// (non-portable size; 16 SMs of one GPC).
//
// What it computes is exactly the three stages of the large path (histogram,
// exclusive scan, count-expansion — PAPER.md:52, 86-92, 168-190, 259-284):
//   1. CTA r builds the compressed histogram of its slice of the keys in shared
//      memory (u16 counters packed two per word; a counter
//      crossing 2^15 is exchanged into the u64 spill, as in hist16.cu);
//   2. every CTA writes its table to L2 (the first step of the two-step merge,
//      PAPER.md:89), cluster barrier; CTA r owns bins [r B, (r+1) B), B = 65536
//      / 16, and sums them over the 16 tables plus the spill.  (Reading the peers'
//      tables through distributed shared memory instead took 7.5 us: DSMEM
//      serves ~20 B/clk per SM, L2 several times that.)
//   3. exclusive scan of its bins, the 16 CTA totals exchanged through
//      distributed shared memory, and the expansion of its bins into the output
//      with 16-byte stores (Alg. 5 with t = 0, l_b = 0).
// Why: at 2^20 keys the two-kernel path (cooperative histogram with two grid
// barriers and 148 x 128 KB partials, then the expansion) is latency-bound
// (29 us); one cluster launch keeps every intermediate on chip.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"

#ifdef FS_SMALL_TRACE  // scripts/microbench/small_trace.cu: %globaltimer per phase, CTA 0 thread 0
__device__ unsigned long long g_small_trace[16][16];
#define FS_STRACE(i)                                                        \
  do {                                                                      \
    if (threadIdx.x == 0) {                                                 \
      unsigned long long t_;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
      g_small_trace[blockIdx.x][i] = t_;                                    \
    }                                                                       \
  } while (0)
#else
#define FS_STRACE(i) \
  do {               \
  } while (0)
#endif

namespace fs {
namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr uint32_t kCluster = 16;
constexpr uint32_t kBinsPerCta = kHistBins / kCluster;      // 4,096
constexpr uint32_t kBinsPerThread = kBinsPerCta / kThreads;  // 4
constexpr uint32_t kHotMask = 0x80008000u;                   // either 16-bit half >= 2^15
#ifndef FS_SMALL_WARM
#define FS_SMALL_WARM 1
#endif
#ifndef FS_SMALL16_MAX_N
#define FS_SMALL16_MAX_N (1ull << 18)  // 2^18: every distribution faster; 2^19: uniform / sorted faster, constant slower
#endif
constexpr uint64_t kSmallMaxN = FS_SMALL16_MAX_N;  // above: the two-kernel path
constexpr uint32_t kStage = kHistBins;    // u16 positions per staging window (the 128 KB table)
constexpr uint32_t kStageRunMax = 64;     // longest run the staging fill takes; longer: the search path

FS_DEVINL uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// 8-byte load from the same shared-memory offset in cluster CTA `rank`
// (distributed shared memory: mapa + ld.shared::cluster).
FS_DEVINL uint2 ld_dsmem_v2(uint32_t laddr, uint32_t rank) {
  uint32_t raddr;
  uint2 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(rank));
  asm volatile("ld.shared::cluster.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(raddr) : "memory");
  return v;
}

__shared__ uint32_t s_spilled;  // this CTA sent a counter to the spill

FS_DEVINL uint32_t ld_dsmem_u32(uint32_t laddr, uint32_t rank) {
  uint32_t raddr, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(raddr) : "memory");
  return v;
}

FS_DEVINL void spill_word(uint32_t* sh, uint32_t w, unsigned long long* spill) {
  const uint32_t x = atomicExch(&sh[w], 0u);
  s_spilled = 1;
  if (x & 0xFFFFu) atomicAdd(&spill[2 * w], (unsigned long long)(x & 0xFFFFu));
  if (x >> 16) atomicAdd(&spill[2 * w + 1], (unsigned long long)(x >> 16));
}

FS_DEVINL void add_key(uint32_t* sh, uint32_t k, unsigned long long* spill) {
  const uint32_t w = k >> 1;
  const uint32_t old = atomicAdd(&sh[w], (k & 1u) ? 0x10000u : 1u);
  if (old & kHotMask) spill_word(sh, w, spill);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_sort16_small(const uint16_t* __restrict__ keys, uint64_t n, uint16_t* __restrict__ out,
                   unsigned long long* __restrict__ spill, uint32_t* __restrict__ partials) {
  extern __shared__ uint4 smem_v4[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem_v4);  // 32,768 words = 65,536 u16 counters
  __shared__ uint32_t pfx[kBinsPerCta + 1];              // first output position of each owned bin
  __shared__ uint32_t wsum[kThreads / 32];
  __shared__ uint32_t cta_total, cta_max;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t r = cl.block_rank();
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t b0 = r * kBinsPerCta;
  FS_STRACE(0);
#if FS_SMALL_WARM
  // Touch every buffer's translation early: each phase's first access to a new
  // buffer would otherwise wait for a TLB fill.
  if (tid < 3) {
    const void* p = tid == 0 ? (const void*)(keys + n * r / kCluster)
                  : tid == 1 ? (const void*)(out + n * r / kCluster) : (const void*)(spill + b0);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
#endif

  // ---- zero the table and this CTA's share of the spill
  for (int i = tid; i < kHistWords / 4; i += kThreads) smem_v4[i] = make_uint4(0, 0, 0, 0);
  for (uint32_t i = tid; i < kBinsPerCta; i += kThreads) spill[b0 + i] = 0;
  if (tid == 0) {
    s_spilled = 0;
    cta_max = 0;
  }
  cl.sync();
  FS_STRACE(1);

  // ---- 1. histogram of the slice [s0, s1)
  const uint64_t s0 = n * r / kCluster, s1 = n * (r + 1) / kCluster;
  const uint64_t a0 = (s0 + 7) & ~(uint64_t)7, a1 = s1 & ~(uint64_t)7;  // 16-byte vectors inside
  const bool vec_ok = (((uintptr_t)keys) & 15) == 0 && a0 < a1;
  if (vec_ok) {
    const uint4* v = reinterpret_cast<const uint4*>(keys + a0);
    const uint64_t nv = (a1 - a0) / 8;
    for (uint64_t i0 = 0; i0 < nv; i0 += kThreads) {  // warp-uniform trip count (vote below)
      const bool valid = i0 + tid < nv;
      const uint4 q = valid ? ld_stream_v4(v + i0 + tid) : make_uint4(0, 0, 0, 0);
      const uint32_t k0 = q.x & 0xFFFFu;
      const bool eq = valid && q.x == q.y && q.y == q.z && q.z == q.w && (q.x >> 16) == k0;
      // a warp whose 256 keys are one value (runs, constant input) adds once
      const uint32_t kl0 = __shfl_sync(kFull, k0, 0);  // every lane, before the vote
      if (__all_sync(kFull, eq && k0 == kl0)) {
        if (lane == 0) {
          const uint32_t w = k0 >> 1;
          const uint32_t old = atomicAdd(&sh[w], (k0 & 1u) ? (256u << 16) : 256u);
          if (old & kHotMask) spill_word(sh, w, spill);
        }
      } else if (valid) {
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          add_key(sh, w4[j] & 0xFFFFu, spill);
          add_key(sh, w4[j] >> 16, spill);
        }
      }
    }
    for (uint64_t i = s0 + tid; i < a0; i += kThreads) add_key(sh, keys[i], spill);
    for (uint64_t i = a1 + tid; i < s1; i += kThreads) add_key(sh, keys[i], spill);
  } else {
    for (uint64_t i = s0 + tid; i < s1; i += kThreads) add_key(sh, keys[i], spill);
  }
  __syncthreads();
  {  // the table to L2 (coalesced 16-byte stores)
    uint4* dst = reinterpret_cast<uint4*>(partials + (uint64_t)r * kHistWords);
    for (int i = tid; i < kHistWords / 4; i += kThreads) dst[i] = smem_v4[i];
  }
  __threadfence();  // the table and the spill adds are visible cluster-wide after the barrier
  cl.sync();
  FS_STRACE(2);

  // ---- 2. merge this CTA's bins over the 16 tables (from L2):
  //         thread t owns bins b0 + 4t .. b0 + 4t + 3 (two counter words)
  uint32_t cnt[kBinsPerThread] = {0, 0, 0, 0};
  {
    static_assert(kBinsPerThread == 4, "two counter words per thread");
    const uint32_t w = (b0 + tid * kBinsPerThread) >> 1;
    // did any CTA spill? (one flag per CTA; the spill is read only then)
    const uint32_t f = lane < kCluster ? ld_dsmem_u32(smem_addr(&s_spilled), lane) : 0u;
    const bool any_spill = __any_sync(kFull, f != 0);
    uint2 x[kCluster];
#pragma unroll
    for (uint32_t c = 0; c < kCluster; ++c)  // 16 loads in flight, coalesced across the threads
      x[c] = __ldcg(reinterpret_cast<const uint2*>(partials + (uint64_t)c * kHistWords + w));
#pragma unroll
    for (uint32_t c = 0; c < kCluster; ++c) {
      cnt[0] += x[c].x & 0xFFFFu;
      cnt[1] += x[c].x >> 16;
      cnt[2] += x[c].y & 0xFFFFu;
      cnt[3] += x[c].y >> 16;
    }
    if (any_spill) {
#pragma unroll
      for (uint32_t j = 0; j < kBinsPerThread; ++j) cnt[j] += (uint32_t)__ldcg(&spill[2 * w + j]);
    }
  }
  uint32_t local = 0, mx = 0;
#pragma unroll
  for (uint32_t j = 0; j < kBinsPerThread; ++j) {
    local += cnt[j];
    mx = max(mx, cnt[j]);
  }
  mx = __reduce_max_sync(kFull, mx);
  if (lane == 0) atomicMax(&cta_max, mx);
  FS_STRACE(9);
  const uint32_t inc = warp_inclusive_scan<uint32_t>(local);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = wsum[lane];
    const uint32_t xi = warp_inclusive_scan<uint32_t>(x);
    wsum[lane] = xi - x;
    if (lane == 31) cta_total = xi;
  }
  __syncthreads();
  {
    uint32_t run = wsum[warp] + inc - local;
#pragma unroll
    for (uint32_t j = 0; j < kBinsPerThread; ++j) {
      pfx[tid * kBinsPerThread + j] = run;
      run += cnt[j];
    }
    if (tid == kThreads - 1) pfx[kBinsPerCta] = run;
  }
  FS_STRACE(3);
  cl.sync();  // every CTA's total is written (and every table has been read)
  FS_STRACE(4);
  uint64_t base = 0;  // this CTA's output start = totals of the lower-ranked CTAs
  for (uint32_t c = 0; c < r; ++c) base += *cl.map_shared_rank(&cta_total, c);
  const uint32_t total = pfx[kBinsPerCta];
  FS_STRACE(7);

  // ---- 3. expansion: global positions [base, base + total), 8 keys per 16-byte store
  const uint64_t g0 = base, g1 = base + total;
  auto bin_at = [&](uint32_t rel) -> uint32_t {  // largest i with pfx[i] <= rel
    uint32_t lo = 0, hi = kBinsPerCta;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pfx[mid] <= rel) lo = mid; else hi = mid;
    }
    return lo;
  };
  const bool aligned = ((uintptr_t)out & 15) == 0;
  if (cta_max <= kStageRunMax) {
    // Short runs (the common case): the runs are written into shared memory by
    // their bins (thread t: bins t, t + 1024, ... so a warp's runs are adjacent),
    // then streamed out in 16-byte stores, 64K positions per window.  (Searching
    // each output vector's bins instead took ~14 us per 64K keys: long chains of
    // dependent shared loads.)
    uint16_t* stage = reinterpret_cast<uint16_t*>(sh);
    for (uint32_t w0 = 0; w0 < total; w0 += kStage) {
      const uint32_t w1 = min(total, w0 + kStage);
#pragma unroll
      for (uint32_t m = 0; m < kBinsPerThread; ++m) {
        const uint32_t v = m * kThreads + tid;
        const uint32_t p = max(pfx[v], w0), e = min(pfx[v + 1], w1);
        for (uint32_t q = p; q < e; ++q) stage[q - w0] = (uint16_t)(b0 + v);
      }
      __syncthreads();
      const uint64_t q0 = g0 + w0, q1 = g0 + w1;  // global positions of the window
      const uint64_t v0 = aligned ? (q0 + 7) / 8 : 0, v1 = aligned ? q1 / 8 : 0;
      for (uint64_t c = v0 + tid; c < v1; c += kThreads) {
        const uint16_t* src = stage + (c * 8 - q0);
        st_stream_v4(reinterpret_cast<uint4*>(out) + c,
                     make_uint4(src[0] | ((uint32_t)src[1] << 16), src[2] | ((uint32_t)src[3] << 16),
                                src[4] | ((uint32_t)src[5] << 16), src[6] | ((uint32_t)src[7] << 16)));
      }
      auto edge = [&](uint64_t a, uint64_t b) {
        for (uint64_t p = a + tid; p < b; p += kThreads) out[p] = stage[p - q0];
      };
      if (v0 < v1) {
        edge(q0, v0 * 8);
        edge(v1 * 8, q1);
      } else {
        edge(q0, q1);
      }
      __syncthreads();  // the stage is refilled by the next window
    }
    FS_STRACE(8);
    FS_STRACE(5);
    cl.sync();  // no CTA leaves while a peer may still read its cta_total
    FS_STRACE(6);
    return;
  }
  const uint64_t c0 = aligned ? (g0 + 7) / 8 : 0, c1 = aligned ? g1 / 8 : 0;  // whole 16-byte chunks
  // A thread's chunks come in increasing order: its bin index only moves forward
  // (a few linear steps, then a binary search from where it is; as expand16.cu).
  auto advance = [&](uint32_t j, uint32_t l) -> uint32_t {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (pfx[j + 1] > l) return j;
      ++j;
    }
    uint32_t lo = j, hi = kBinsPerCta;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pfx[mid] <= l) lo = mid; else hi = mid;
    }
    return lo;
  };
  uint32_t j = 0;
  for (uint64_t c = c0 + tid; c < c1; c += kThreads) {
    const uint32_t l = (uint32_t)(c * 8 - g0);
    j = advance(j, l);
    uint32_t run_end = pfx[j + 1];
    uint32_t packed[4];
    if (l + 7 < run_end) {  // the whole vector lies in one run (the dense case)
      const uint32_t v = b0 + j;
      packed[0] = packed[1] = packed[2] = packed[3] = v | (v << 16);
    } else {
      uint32_t jj = j;
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        uint32_t pair = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (l + e + h >= run_end) {
            jj = advance(jj, l + e + h);
            run_end = pfx[jj + 1];
          }
          pair |= (b0 + jj) << (16 * h);
        }
        packed[e / 2] = pair;
      }
    }
    st_stream_v4(reinterpret_cast<uint4*>(out) + c, make_uint4(packed[0], packed[1], packed[2], packed[3]));
  }
  FS_STRACE(8);
  // positions outside whole chunks (the edges, or everything if out is unaligned)
  auto scalar = [&](uint64_t p0, uint64_t p1) {
    for (uint64_t p = p0 + tid; p < p1; p += kThreads) out[p] = (uint16_t)(b0 + bin_at((uint32_t)(p - g0)));
  };
  if (c0 < c1) {
    scalar(g0, c0 * 8);
    scalar(c1 * 8, g1);
  } else {
    scalar(g0, g1);
  }
  FS_STRACE(5);
  cl.sync();  // no CTA leaves while a peer may still read its cta_total
  FS_STRACE(6);
}

}  // namespace

uint64_t small16_max_n() { return kSmallMaxN; }

cudaError_t launch_sort16_small(const uint16_t* keys, uint64_t n, uint16_t* out, unsigned long long* spill,
                                uint32_t* partials, cudaStream_t s) {
  constexpr int smem = kHistWords * 4;  // 128 KB table (+ 16 KB static: the prefix)
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_sort16_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_sort16_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCluster);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_sort16_small, keys, n, out, spill, partials);
}

}  // namespace fs
