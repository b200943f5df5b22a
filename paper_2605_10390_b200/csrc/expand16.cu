// expand16.cu — stage 3 of the u16 path: count-expansion (G3).
//
// What it computes: Alg. 5 ReconstructAll (§III.G.3) with
// t = p - l_n = 0 and l_b = 0 — the entries carry no bits, so bin b is emitted
// C[b] times in ascending b ("if C[b] = 0 continue").  Written as
// a function of output position j: out[j] = the v with P[v] <= j < P[v+1].
// Restricted to global positions [out_begin, out_end) so a rank of the
// multi-GPU path writes only its own range (SURVEY.md §8(e) Mode B).
//
// The prefix P comes in one of two forms:
//  * global (fs_expand_u16): P[0..nbins] as given by the caller;
//  * two-level (the fused sort): P[v] = L[v] + B[v >> 9] where L holds the
//    slice-local exclusive prefixes written by the histogram kernel and B the
//    exclusive scan of its 128 slice totals, computed here by every CTA (the
//    last step of GetIndex, Alg. 3, folded into this kernel's first search
//    round, so the histogram kernel needs no cross-slice pass).
//
// B200 design: HBM-write bound (2 B per key).
// Each CTA owns an output tile of 32,768 keys (64 KB).  The first and last bin
// touching the tile are found by a block-parallel search (L2-resident data):
// one round over 256 coarse points (global form) or the 128 slice bases
// (two-level form), one round over the <= 512 points between them
// (__syncthreads_count does the comparisons).  The tile's slice of P is staged
// in shared memory as 32-bit offsets relative to the tile; each thread emits 8
// keys per 16-byte streaming store (consecutive lanes -> consecutive 16 B) and
// tracks its current run monotonically (its positions only increase).  The
// kernel is launched with programmatic dependent launch so its launch overlaps
// the histogram kernel's tail.  Unaligned head/tail keys: CTA 0, one per thread.
#include "common.cuh"
#include "kernels.cuh"

#ifdef FS_EXPAND_TRACE
// Debug-only per-CTA timestamps (scripts/microbench/expand_trace.cu builds this
// file with -DFS_EXPAND_TRACE); compiled out of libfractalsort.so.
__device__ unsigned long long g_expand_trace[1 << 16][4];
#define FS_XTRACE(i)                                                          \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < (1u << 16)) {                        \
      unsigned long long t_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_expand_trace[blockIdx.x][i] = t_;                                     \
      unsigned smid_;                                                         \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                      \
      g_expand_trace[blockIdx.x][3] = smid_;                                  \
    }                                                                         \
  } while (0)
#else
#define FS_XTRACE(i) \
  do {               \
  } while (0)
#endif

namespace fs {
namespace {

#ifndef FS_EXPAND_THREADS
#define FS_EXPAND_THREADS 256
#endif
constexpr int kThreads = FS_EXPAND_THREADS;
#ifndef FS_EXPAND_VPT
#define FS_EXPAND_VPT 16
#endif
constexpr int kVecPerThread = FS_EXPAND_VPT;                       // max 16-byte vectors per thread
constexpr int kSliceCap = 4096;                                    // staged P entries
#ifndef FS_EXPAND_SLICE_STAGE
#define FS_EXPAND_SLICE_STAGE 1  // two-level prefix: stage whole slices in one round trip (0: search first)
#endif
constexpr int kSliceShift = 9;                                     // two-level: 512-bin slices
constexpr int kNumSlices = 65536 >> kSliceShift;                   // 128
static_assert(kNumSlices == kHistSlices, "slice layout shared with hist16.cu");

// P[v] for v in [0, nbins]: global array, or slice-local prefix + slice base.
template <bool kTwoLevel>
struct PrefixView {
  const uint64_t* P;          // global P[0..nbins] or slice-local L[0..nbins)
  const uint64_t* base;       // two-level: shared-memory B[0..128] (B[128] = total)
  uint64_t nbins;
  FS_DEVINL uint64_t operator()(uint64_t v) const {
    if (!kTwoLevel) return __ldcg(P + v);
    return v >= nbins ? base[kNumSlices] : __ldcg(P + v) + base[v >> kSliceShift];
  }
  // P at a coarse-grid point; two-level grid points are slice starts (L = 0 there).
  FS_DEVINL uint64_t coarse(uint64_t v) const {
    if (!kTwoLevel) return __ldcg(P + v);
    return base[v >> kSliceShift];
  }
};

// Thread-level binary search: largest v in [lo, hi) with P(v) <= o, given P(lo) <= o.
template <class View>
FS_DEVINL uint64_t thread_last_le(const View& P, uint64_t lo, uint64_t hi, uint64_t o) {
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (P(mid) <= o) lo = mid; else hi = mid;
  }
  return lo;
}

// Largest j in [j0, hi) with rel[j] <= l, given rel[j0] <= l: a short linear
// probe (runs are usually long) then binary search.
FS_DEVINL uint32_t advance(const uint32_t* rel, uint32_t j, uint32_t hi, uint32_t l) {
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (j + 1 >= hi || rel[j + 1] > l) return j;
    ++j;
  }
  uint32_t lo = j;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rel[mid] <= l) lo = mid; else hi = mid;
  }
  return lo;
}

// Block-wide: largest v < nbins with P(v) <= o for two positions at once, in two
// rounds: a coarse grid of `cs`-spaced points, then the points between them.
template <class View>
FS_DEVINL void block_last_le2(const View& P, uint64_t nbins, uint64_t cs, uint64_t o_a, uint64_t o_b,
                              uint64_t& v_a, uint64_t& v_b) {
  const uint32_t tid = threadIdx.x;
  const uint64_t ci = (uint64_t)tid * cs;
  const uint64_t p = ci < nbins ? P.coarse(ci) : ~0ull;
  const uint64_t c_a = (uint64_t)__syncthreads_count(p <= o_a) - 1;  // P(0) = 0 <= o
  const uint64_t c_b = (uint64_t)__syncthreads_count(p <= o_b) - 1;
  uint32_t n_a = 0, n_b = 0;
  for (uint64_t j = tid; j < cs; j += kThreads) {  // cs <= 512: at most two rounds per thread
    const uint64_t fa = c_a * cs + j, fb = c_b * cs + j;
    n_a += fa < nbins && P(fa) <= o_a;
    n_b += fb < nbins && P(fb) <= o_b;
  }
  __shared__ uint32_t cnt_sh[2];
  if (tid == 0) cnt_sh[0] = cnt_sh[1] = 0;
  __syncthreads();
  if (n_a) atomicAdd(&cnt_sh[0], n_a);
  if (n_b) atomicAdd(&cnt_sh[1], n_b);
  __syncthreads();
  v_a = c_a * cs + cnt_sh[0] - 1;
  v_b = c_b * cs + cnt_sh[1] - 1;
}

// kVpt: vectors per thread, fixed at compile time (16) for large outputs; 0 means
// the runtime value `vpt` (small outputs, smaller tiles).
template <bool kTwoLevel, int kVpt>
#ifndef FS_EXPAND_MINB
#define FS_EXPAND_MINB (2048 / FS_EXPAND_THREADS)  // CTAs per SM the register budget is sized for (32 registers)
#endif
__global__ void __launch_bounds__(kThreads, FS_EXPAND_MINB)
    k_expand16(const uint64_t* __restrict__ P, const uint64_t* __restrict__ slice_tot, uint64_t nbins, uint64_t pos0,
               uint64_t nvec, uint16_t* __restrict__ out_body, uint64_t out_begin, uint64_t head, uint64_t tail_pos,
               uint64_t tail_n, uint16_t* __restrict__ out, uint32_t vpt_rt) {
  const uint32_t vpt = kVpt ? (uint32_t)kVpt : vpt_rt;
  __shared__ uint32_t rel[kSliceCap];
  __shared__ uint32_t zeros_sh;
  __shared__ uint64_t base_sh[kNumSlices + 1];
  const uint32_t tid = threadIdx.x;
  // Programmatic dependent launch: everything above overlaps the producer's tail;
  // P is read only after the producer grid has completed.
  cudaGridDependencySynchronize();
  FS_XTRACE(0);
  if (threadIdx.x == 0) zeros_sh = 0;  // (first read after the setup's barriers)

#ifndef FS_EXPAND_WARP_SETUP
#define FS_EXPAND_WARP_SETUP 0
#endif
  if (kTwoLevel && FS_EXPAND_WARP_SETUP) {  // slice bases: exclusive scan of the 128 slice totals, by warp 0
    if (tid < 32) {
      uint64_t t[4], run = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] = __ldcg(slice_tot + tid * 4 + i);
#pragma unroll
      for (int i = 0; i < 4; ++i) run += t[i];
      uint64_t ex = warp_inclusive_scan<uint64_t>(run) - run;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        base_sh[tid * 4 + i] = ex;
        ex += t[i];
      }
      if (tid == 31) base_sh[kNumSlices] = ex;
    }
    __syncthreads();
  } else if (kTwoLevel) {  // slice bases: exclusive scan of the 128 slice totals (4 warps)
    __shared__ uint64_t wtot[kThreads / 32];
    const uint64_t t = tid < kNumSlices ? __ldcg(slice_tot + tid) : 0ull;
    const uint64_t inc = warp_inclusive_scan<uint64_t>(t);
    if ((tid & 31) == 31) wtot[tid >> 5] = inc;
    __syncthreads();
    uint64_t off = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      if (w < (int)(tid >> 5)) off += wtot[w];
      all += wtot[w];
    }
    if (tid < kNumSlices) base_sh[tid] = off + inc - t;
    if (tid == 0) base_sh[kNumSlices] = all;
    __syncthreads();
  }
  static_assert(kNumSlices == 4 * 32, "warp 0 scans the slice totals four per lane");
  const PrefixView<kTwoLevel> Pv{P, base_sh, nbins};

  // Unaligned head/tail keys (< 8 each): one per thread in CTA 0.
  if (blockIdx.x == 0 && tid < head + tail_n) {
    const uint64_t j = tid < head ? out_begin + tid : tail_pos + (tid - head);
    out[j - out_begin] = (uint16_t)thread_last_le(Pv, 0, nbins, j);
  }
  if (nvec == 0) return;

  const uint64_t tile_vec = (uint64_t)kThreads * vpt;  // vectors per tile (vpt <= kVecPerThread)
#ifndef FS_EXPAND_TILE_ORDER
#define FS_EXPAND_TILE_ORDER 1
#endif
  // Tile order: CTAs b = 0, 1, 2, 3, ... take tiles 0, G-1, 1, G-2, ...  The
  // slowest tiles of skewed inputs are the sparse ends of the key range (many
  // short runs: Gauss tile 0 and G-1 take ~3x a dense tile, expand_trace.cu);
  // dispatched first, they finish inside the first wave instead of extending
  // the last one.  (Rotating only the last 16-256 tiles to the front instead:
  // Gauss the same, Zipf 5 us slower -- profiles/r02/u16_variants_expand_order.txt.)
  const uint64_t tile = FS_EXPAND_TILE_ORDER ? ((blockIdx.x & 1u) ? gridDim.x - 1u - (blockIdx.x >> 1) : (blockIdx.x >> 1))
                                             : blockIdx.x;
  const uint64_t vec0 = tile * tile_vec;
  const uint64_t vec_end = vec0 + tile_vec < nvec ? vec0 + tile_vec : nvec;
  const uint64_t o0 = pos0 + vec0 * 8;  // first global position of the tile
  const uint32_t len = (uint32_t)((vec_end - vec0) * 8);
  uint64_t v_lo = 0, v_hi = 0, m = 0;
  uint4* dst = reinterpret_cast<uint4*>(out_body) + vec0;
  bool staged = false;
  if (kTwoLevel && FS_EXPAND_SLICE_STAGE) {
    // One L2 round trip: the slices holding the tile's first and last position
    // follow from the bases in shared memory; all their bins are staged at once
    // (the bins before the tile stage as 0 and are skipped by the first search).
    uint32_t sa, sb;
    if (FS_EXPAND_WARP_SETUP) {  // every warp finds them itself from the bases (ballots), no block barrier
      const uint32_t lane = tid & 31u;
      uint32_t ca = 0, cbn = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t b = base_sh[lane * 4 + i];
        ca += __popc(__ballot_sync(kFull, b <= o0));
        cbn += __popc(__ballot_sync(kFull, b <= o0 + len - 1));
      }
      sa = ca - 1;
      sb = cbn - 1;
    } else {
      sa = (uint32_t)__syncthreads_count(tid < kNumSlices && base_sh[tid] <= o0) - 1;
      sb = (uint32_t)__syncthreads_count(tid < kNumSlices && base_sh[tid] <= o0 + len - 1) - 1;
    }
    const uint32_t nb = (sb - sa + 1) << kSliceShift;
    if (nb < (uint32_t)kSliceCap) {
      v_lo = (uint64_t)sa << kSliceShift;
      m = nb + 1;
      uint32_t z = 0;
      for (uint32_t j = tid; j < nb; j += kThreads) {
        const uint64_t p = __ldcg(P + v_lo + j) + base_sh[sa + (j >> kSliceShift)];
        rel[j] = p <= o0 ? 0u : (p - o0 >= len ? len : (uint32_t)(p - o0));
        z += p <= o0;
      }
      // the bins before the tile stage as 0 (a prefix): every thread's search
      // starts at the last of them instead of at 0
      if (z) atomicAdd(&zeros_sh, z);
      if (tid == 0) {  // sentinel: P at the first bin of slice sb + 1 (or n)
        const uint64_t p = base_sh[sb + 1];
        rel[nb] = p - o0 >= len ? len : (uint32_t)(p - o0);
      }
      staged = true;
    }
  }
  if (!staged) {
    // Coarse grid: the 128 slice starts (two-level: their P values are the bases
    // already in shared memory) or 256 evenly spaced points of the global P.
    block_last_le2(Pv, nbins, kTwoLevel ? (uint64_t)1 << kSliceShift : (nbins + kThreads - 1) / kThreads, o0,
                   o0 + len - 1, v_lo, v_hi);
    m = v_hi - v_lo + 2;  // P[v_lo .. v_hi+1]
    if (m <= (uint64_t)kSliceCap) {
      for (uint32_t j = tid; j < m; j += kThreads) {
        const uint64_t p = Pv(v_lo + j);
        rel[j] = p <= o0 ? 0u : (p - o0 >= len ? len : (uint32_t)(p - o0));
      }
      staged = true;
    }
  }

  if (staged) {
    __syncthreads();
    FS_XTRACE(1);
    const uint32_t hi = (uint32_t)m - 1;  // searches stay below the sentinel rel[m-1] >= len
#ifndef FS_EXPAND_ZSTART
#define FS_EXPAND_ZSTART 1
#endif
    uint32_t j = FS_EXPAND_ZSTART && zeros_sh ? zeros_sh - 1 : 0;  // rel[j] = 0: a valid start for every position
#pragma unroll 4
    for (uint32_t k = 0; k < vpt; ++k) {
      const uint32_t q = k * kThreads + tid;
      const uint32_t l = q * 8;
      if (l >= len) break;
      j = advance(rel, j, hi, l);
      uint32_t run_end = rel[j + 1];
      uint32_t packed[4];
      if (l + 7 < run_end) {  // the whole vector lies in one run (common case)
        const uint32_t v = (uint32_t)(v_lo + j);
        const uint32_t pv = v | (v << 16);
        packed[0] = packed[1] = packed[2] = packed[3] = pv;
      } else {
#ifndef FS_EXPAND_ONE_BOUNDARY
#define FS_EXPAND_ONE_BOUNDARY 1
#endif
        uint32_t jj = j;
        const uint32_t je = FS_EXPAND_ONE_BOUNDARY ? advance(rel, j, hi, l + 7) : 0u;  // bin of the last key
        if (FS_EXPAND_ONE_BOUNDARY && rel[je] == run_end) {
          // one boundary (the bins between j and je are empty): keys before
          // run_end are bin j, the rest bin je -- branch-free, so a warp whose
          // lanes straddle runs of ~100 keys (Zipf) does not serialise on the
          // per-key loop below
          const uint32_t va = (uint32_t)(v_lo + j) & 0xFFFFu, vb = (uint32_t)(v_lo + je) & 0xFFFFu;
#pragma unroll
          for (int e = 0; e < 8; e += 2)
            packed[e / 2] = (l + e < run_end ? va : vb) | ((l + e + 1 < run_end ? va : vb) << 16);
        } else {
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            uint32_t pair = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t pos = l + e + h;
              if (pos >= run_end) {
                jj = advance(rel, jj, hi, pos);
                run_end = rel[jj + 1];
              }
              pair |= ((uint32_t)(v_lo + jj) & 0xFFFFu) << (16 * h);
            }
            packed[e / 2] = pair;
          }
        }
      }
      st_stream_v4(dst + q, make_uint4(packed[0], packed[1], packed[2], packed[3]));
    }
    __syncthreads();
    FS_XTRACE(2);
  } else {
    // Very sparse tile (more than kSliceCap bins): search P in L2 per position.
#pragma unroll 1
    for (uint32_t k = 0; k < vpt; ++k) {
      const uint32_t q = k * kThreads + tid;
      const uint32_t l = q * 8;
      if (l >= len) break;
      uint32_t packed[4] = {0, 0, 0, 0};
      uint64_t v = thread_last_le(Pv, v_lo, v_hi + 1, o0 + l);
      uint64_t run_end = Pv(v + 1);
      for (int e = 0; e < 8; ++e) {
        const uint64_t pos = o0 + l + e;
        if (pos >= run_end) {
          v = thread_last_le(Pv, v + 1, v_hi + 1, pos);
          run_end = Pv(v + 1);
        }
        packed[e / 2] |= ((uint32_t)v & 0xFFFFu) << (16 * (e & 1));
      }
      st_stream_v4(dst + q, make_uint4(packed[0], packed[1], packed[2], packed[3]));
    }
  }
}

template <bool kTwoLevel>
cudaError_t launch(const uint64_t* prefix, const uint64_t* slice_tot, uint64_t nbins, uint64_t out_begin,
                   uint64_t out_end, uint16_t* out, cudaStream_t s) {
  const uint64_t n = out_end - out_begin;
  if (n == 0) return cudaSuccess;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(out);
  uint64_t head = ((16 - (addr & 15)) & 15) / 2;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 8;
  const uint64_t tail_n = n - head - nvec * 8;
  const uint64_t pos0 = out_begin + head;
  const uint64_t tail_pos = pos0 + nvec * 8;
  // 64 KB tiles for large outputs; smaller tiles so that small outputs still
  // give every SM several CTAs.
  const uint64_t want = (uint64_t)device_info().sm_count * 4;
  uint32_t vpt = kVecPerThread;
  while (vpt > 1 && (nvec + (uint64_t)kThreads * vpt - 1) / ((uint64_t)kThreads * vpt) < want) vpt >>= 1;
  uint64_t grid = (nvec + (uint64_t)kThreads * vpt - 1) / ((uint64_t)kThreads * vpt);
  if (grid == 0) grid = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  uint16_t* body = out + head;
  if (vpt == kVecPerThread)
    return cudaLaunchKernelEx(&cfg, k_expand16<kTwoLevel, kVecPerThread>, prefix, slice_tot, nbins, pos0, nvec, body,
                              out_begin, head, tail_pos, tail_n, out, vpt);
  return cudaLaunchKernelEx(&cfg, k_expand16<kTwoLevel, 0>, prefix, slice_tot, nbins, pos0, nvec, body, out_begin, head,
                            tail_pos, tail_n, out, vpt);
}

}  // namespace

cudaError_t launch_expand16(const uint64_t* prefix, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                            uint16_t* out, cudaStream_t s) {
  return launch<false>(prefix, nullptr, nbins, out_begin, out_end, out, s);
}

cudaError_t launch_expand16_two_level(const uint64_t* slice_prefix, const uint64_t* slice_tot, uint64_t out_begin,
                                      uint64_t out_end, uint16_t* out, cudaStream_t s) {
  return launch<true>(slice_prefix, slice_tot, kHistBins, out_begin, out_end, out, s);
}

}  // namespace fs
