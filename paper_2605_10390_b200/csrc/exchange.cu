// exchange.cu — the distributed pair sort's exact splitters and its fused
// partition-to-peer exchange (SURVEY.md §8(e) pairs, §8(f) NEXT-2).
//
// Splitters by compressed histograms, no sampling (PAPER.md:95 Fractal RMW,
// 168-190 GetIndex; ledger 13, 23).  Rank d owns global positions
// [s_d, s_{d+1}), s_d = floor(dN/G).  The key K_d of the element at position
// s_d is found digit by digit, 16 bits at a time from the top: level 1 is the
// histogram of the top digit over every key of every rank (fs_histogram16_u64,
// all-reduced), which fixes the top digit of every K_d and how many keys lie
// below it; each later level is the histogram of the next digit over the keys
// that share K_d's digits so far (fs_digit_counts_sorted_u64 on the locally
// sorted candidates, all-reduced).  Four levels fix a 64-bit K_d exactly.
//
// The fused exchange (fs_pair_classes_u64 + fs_pair_scatter_u64_u32): every
// element gets a class -- 2d for K_{d-1} < key < K_d, 2d + 1 for key == K_d
// (the lowest such d) -- and the rank's elements in class order (stable within
// a class) form a sequence in which every owner's share is ONE contiguous
// range [cut_d, cut_{d+1}) (ties at a splitter are split by the caller's cuts:
// lower rank first, then input order).  The scatter writes each
// (key, value) straight to bases[d] + (Q - cut_d) in owner d's receive buffer
// (CUDA IPC peer memory over NVLink), Q its class-order index: one pass over
// the rank's pairs, no local sort before the exchange, no staging buffer and no
// all-to-all; the owner then sorts what arrived once.
#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 1024;

// ---------------------------------------------------------------- level-1 histogram
// hist[(key >> shift) & (2^width - 1)] over all keys: per-SM packed u16 counters
// (128 KB of shared memory, two per word as in hist16.cu) with the same spill
// rule -- an add whose returned word has a half >= 2^15 exchanges the word into
// the u64 spill at once; every add is 1 (or one warp's 64 equal digits), so a
// counter stays below 2^15 + 1024 * 2 + 64 < 65,536.
constexpr uint32_t kHot = 0x80008000u;

FS_DEVINL void h_add(uint32_t* sh, uint32_t b, uint32_t cnt, unsigned long long* spill) {
  const uint32_t old = atomicAdd(&sh[b >> 1], (b & 1u) ? (cnt << 16) : cnt);
  if (old & kHot) {
    const uint32_t x = atomicExch(&sh[b >> 1], 0u);
    if (x & 0xFFFFu) atomicAdd(&spill[b & ~1u], (unsigned long long)(x & 0xFFFFu));
    if (x >> 16) atomicAdd(&spill[b | 1u], (unsigned long long)(x >> 16));
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_digit_hist(const uint64_t* __restrict__ keys, uint64_t n, int shift, uint32_t mask,
                 uint32_t* __restrict__ partials, unsigned long long* __restrict__ spill) {
  extern __shared__ uint4 sm4[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(sm4);
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  for (int i = tid; i < kHistWords / 4; i += kThreads) sm4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // grid-strided over pairs of keys (one 16-byte vector when aligned)
  const uint64_t npair = n / 2;
  const bool aligned = ((uintptr_t)keys & 15) == 0;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kThreads; i0 < npair; i0 += (uint64_t)gridDim.x * kThreads) {
    const uint64_t i = i0 + tid;
    uint32_t b0 = 0, b1 = 0;
    const bool valid = i < npair;
    if (valid) {
      uint64_t k0, k1;
      if (aligned) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(keys) + i);
        k0 = ((uint64_t)q.y << 32) | q.x;
        k1 = ((uint64_t)q.w << 32) | q.z;
      } else {
        k0 = __ldcs(keys + 2 * i);
        k1 = __ldcs(keys + 2 * i + 1);
      }
      b0 = (uint32_t)(k0 >> shift) & mask;
      b1 = (uint32_t)(k1 >> shift) & mask;
    }
    // a warp whose 64 digits are all equal adds them with one atomic (runs / constant keys)
    const uint32_t ref = __shfl_sync(kFull, b0, 0);
    if (__all_sync(kFull, valid && b0 == ref && b1 == ref)) {
      if (lane == 0) h_add(sh, ref, 64u, spill);
    } else if (valid) {
      h_add(sh, b0, 1u, spill);
      h_add(sh, b1, 1u, spill);
    }
  }
  if (blockIdx.x == 0 && tid == 0 && (n & 1)) h_add(sh, (uint32_t)(keys[n - 1] >> shift) & mask, 1u, spill);
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(partials + (uint64_t)blockIdx.x * kHistWords);
  for (int i = tid; i < kHistWords / 4; i += kThreads) dst[i] = sm4[i];
}

// ---------------------------------------------------------------- candidates
// Appends (in no particular order) every key whose digit is one of bins[0..nb).
__global__ void __launch_bounds__(256)
    k_select_bins(const uint64_t* __restrict__ keys, uint64_t n, int shift, uint32_t mask,
                  const uint32_t* __restrict__ bins, int nb, uint64_t* __restrict__ out, uint64_t cap,
                  unsigned long long* __restrict__ count) {
  __shared__ uint32_t sb[64];
  if (threadIdx.x < nb) sb[threadIdx.x] = bins[threadIdx.x];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    uint64_t k = 0;
    bool hit = false;
    if (i < n) {
      k = __ldcs(keys + i);
      const uint32_t d = (uint32_t)(k >> shift) & mask;
      for (int j = 0; j < nb; ++j) hit |= d == sb[j];
    }
    const uint32_t m = __ballot_sync(kFull, hit);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, 0);
    const uint64_t at = base + __popc(m & lanemask_lt());
    if (hit && at < cap) out[at] = k;
  }
}

// ---------------------------------------------------------------- level histograms on sorted keys
// hist[j][v] = #{i : (sorted[i] >> shift) == (prefixes[j] >> shift) | v}, v < 2^width:
// two binary searches per (j, v) on the shifted keys (ascending because the keys are).
__global__ void __launch_bounds__(256)
    k_digit_counts_sorted(const uint64_t* __restrict__ sorted, uint64_t m, const uint64_t* __restrict__ prefixes,
                          int np, int shift, int width, uint64_t* __restrict__ hist) {
  const uint64_t nv = 1ull << width;
  const uint64_t idx = blockIdx.x * 256ull + threadIdx.x;
  if (idx >= nv * (uint64_t)np) return;
  const int j = (int)(idx / nv);
  const uint64_t v = idx % nv;
  const uint64_t t = (shift >= 64 ? 0 : (prefixes[j] >> shift)) | v;
  uint64_t lo = 0, hi = m;  // lower bound: first i with (sorted[i] >> shift) >= t
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if ((__ldg(sorted + mid) >> shift) < t) lo = mid + 1; else hi = mid;
  }
  uint64_t lo2 = lo, hi2 = m;  // upper bound: first i with (sorted[i] >> shift) > t
  while (lo2 < hi2) {
    const uint64_t mid = lo2 + (hi2 - lo2) / 2;
    if ((__ldg(sorted + mid) >> shift) <= t) lo2 = mid + 1; else hi2 = mid;
  }
  hist[(uint64_t)j * nv + v] = lo2 - lo;
}

// ---------------------------------------------------------------- classes and the scatter
constexpr int kTileThreads = 256;
constexpr int kPerThread = 8;
constexpr int kTile = kTileThreads * kPerThread;  // 2,048 pairs per tile
constexpr int kMaxG = 16;
constexpr int kMaxClasses = 2 * kMaxG - 1;

// class of a key: 2 * #{j : K_j < key} (+1 when key == K_that)
FS_DEVINL uint32_t key_class(uint64_t k, const uint64_t* K, int nk) {
  int d = 0;
  while (d < nk && K[d] < k) ++d;
  return 2u * d + (d < nk && K[d] == k ? 1u : 0u);
}

__global__ void __launch_bounds__(kTileThreads)
    k_class_counts(const uint64_t* __restrict__ keys, uint64_t n, const uint64_t* __restrict__ splitters, int G,
                   uint64_t* __restrict__ counts, uint64_t T) {
  __shared__ uint64_t K[kMaxG];
  __shared__ uint32_t cnt[kMaxClasses];
  const int C = 2 * G - 1;
  if (threadIdx.x < G - 1) K[threadIdx.x] = splitters[threadIdx.x];
  if (threadIdx.x < C) cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t e0 = blockIdx.x * (uint64_t)kTile;
  for (int i = 0; i < kPerThread; ++i) {
    const uint64_t e = e0 + (uint64_t)i * kTileThreads + threadIdx.x;  // coalesced; counts need no order
    if (e < n) atomicAdd(&cnt[key_class(__ldcs(keys + e), K, G - 1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < C) counts[(uint64_t)threadIdx.x * T + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void k_class_totals(const uint64_t* __restrict__ off, uint64_t T, int C, uint64_t* __restrict__ tot) {
  const int c = threadIdx.x;
  if (c < C) tot[c] = off[(uint64_t)(c + 1) * T] - off[(uint64_t)c * T];
}

struct ScatterArgs {
  const uint64_t* keys;
  const uint32_t* vals;
  uint64_t n, T;
  const uint64_t* splitters;
  int G;
  const uint64_t* off;     // exclusive scan of counts[c * T + t]
  const uint64_t* cuts;    // G + 1 class-order cut points (cuts[0] = 0, cuts[G] = n)
  const uint64_t* bases;   // G: this rank's first slot in owner d's buffer
  uint64_t* const* dkeys;  // G owner key buffers
  uint32_t* const* dvals;  // G owner value buffers
};

// Per tile: classes of its 2,048 pairs (8 consecutive per thread, so the
// per-thread counts scanned over the threads give stable in-tile ranks), the
// pairs staged in shared memory in class order, then written out: consecutive
// threads take consecutive class-order slots, so a warp's stores are runs of
// consecutive addresses of one owner's buffer.
__global__ void __launch_bounds__(kTileThreads) k_class_scatter(ScatterArgs a) {
  __shared__ uint64_t K[kMaxG];
  __shared__ uint64_t cut[kMaxG + 1], base[kMaxG];
  __shared__ uint16_t tcnt[kMaxClasses][kTileThreads];  // per-thread counts -> exclusive in-tile prefixes
  __shared__ uint32_t cstart[kMaxClasses + 1];            // tile's class segments in the staging buffer
  __shared__ uint64_t qbase[kMaxClasses];                 // class-order index of the segment's first pair
  __shared__ uint64_t sk[kTile];
  __shared__ uint32_t sv[kTile];
  __shared__ uint8_t scls[kTile];
  const int G = a.G, C = 2 * G - 1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < G - 1) K[tid] = a.splitters[tid];
  if (tid <= G) cut[tid] = a.cuts[tid];
  if (tid < G) base[tid] = a.bases[tid];
  for (int c = 0; c < C; ++c) tcnt[c][tid] = 0;
  __syncthreads();
  const uint64_t e0 = blockIdx.x * (uint64_t)kTile + (uint64_t)tid * kPerThread;
  uint64_t k[kPerThread];
  uint32_t v[kPerThread], cls[kPerThread];
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    const uint64_t e = e0 + i;
    cls[i] = 0xFFu;
    if (e < a.n) {
      k[i] = __ldcs(a.keys + e);
      v[i] = __ldcs(a.vals + e);
      cls[i] = key_class(k[i], K, G - 1);
      ++tcnt[cls[i]][tid];
    }
  }
  __syncthreads();
  // exclusive scan of every class's 256 per-thread counts (warp w: classes w, w+8, ...)
  for (int c = warp; c < C; c += kTileThreads / 32) {
    uint32_t s[8], run = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] = run;
      run += tcnt[c][lane * 8 + i];
    }
    const uint32_t inc = warp_inclusive_scan<uint32_t>(run);
#pragma unroll
    for (int i = 0; i < 8; ++i) tcnt[c][lane * 8 + i] = (uint16_t)(inc - run + s[i]);
    if (lane == 31) cstart[c + 1] = inc;  // class total in the tile (scanned below)
  }
  __syncthreads();
  if (tid == 0) {
    cstart[0] = 0;
    for (int c = 0; c < C; ++c) cstart[c + 1] += cstart[c];
  }
  if (tid < C) qbase[tid] = a.off[(uint64_t)tid * a.T + blockIdx.x];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    if (cls[i] == 0xFFu) continue;
    const uint32_t c = cls[i];
    const uint32_t r = tcnt[c][tid]++;  // this thread's running in-class rank (own column: no race)
    const uint32_t L = cstart[c] + r;
    sk[L] = k[i];
    sv[L] = v[i];
    scls[L] = (uint8_t)c;
  }
  __syncthreads();
  const uint32_t m = cstart[C];
  for (uint32_t L = tid; L < m; L += kTileThreads) {
    const uint32_t c = scls[L];
    const uint64_t Q = qbase[c] + (L - cstart[c]);
    int d = 0;
    while (d + 1 < G && cut[d + 1] <= Q) ++d;
    const uint64_t slot = base[d] + (Q - cut[d]);
    a.dkeys[d][slot] = sk[L];
    a.dvals[d][slot] = sv[L];
  }
}

size_t round_scan_temp(uint64_t nbins) { return fs_exclusive_scan_u64_temp_bytes(nbins); }

}  // namespace

struct ClassLayout {
  uint64_t T = 0;
  size_t counts = 0, off = 0, stemp = 0, stemp_bytes = 0, cuts = 0, bases = 0, dptr = 0, total = 0;
};

ClassLayout class_layout(uint64_t n, int G) {
  ClassLayout L;
  L.T = (n + kTile - 1) / kTile;
  const uint64_t ne = (uint64_t)(2 * G - 1) * (L.T ? L.T : 1);
  size_t o = 0;
  L.counts = o;
  o = align_up(o + sizeof(uint64_t) * ne);
  L.off = o;
  o = align_up(o + sizeof(uint64_t) * (ne + 1));
  L.stemp = o;
  L.stemp_bytes = round_scan_temp(ne);
  o = align_up(o + L.stemp_bytes);
  L.cuts = o;
  o = align_up(o + sizeof(uint64_t) * (G + 1));
  L.bases = o;
  o = align_up(o + sizeof(uint64_t) * G);
  L.dptr = o;
  o = align_up(o + sizeof(void*) * 2 * G);
  L.total = o;
  return L;
}

}  // namespace fs

using namespace fs;

extern "C" {

size_t fs_histogram16_u64_temp_bytes(uint64_t n) {
  const int grid = hist16_grid(n);
  return align_up(sizeof(uint64_t) * kHistBins) + align_up(sizeof(uint32_t) * kHistWords * (size_t)grid);
}

fs_status fs_histogram16_u64(const uint64_t* keys, uint64_t n, int shift, int width, uint64_t* hist, void* temp,
                             size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (width < 1 || width > 16 || shift < 0 || shift + width > 64)
    return fail(FS_ERR_INVALID_ARGUMENT, "digit [shift %d, +%d) outside a u64 key or wider than 16 bits", shift,
                width);
  if (!hist) return fail(FS_ERR_INVALID_ARGUMENT, "NULL hist");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nb = 1ull << width;
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint64_t) * nb, s);
    return e == cudaSuccess ? finish(s, "fs_histogram16_u64") : cuda_fail(e, "fs_histogram16_u64: memset");
  }
  if (!keys || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  if (((uintptr_t)keys & 7) || ((uintptr_t)hist & 7)) return fail(FS_ERR_INVALID_ARGUMENT, "misaligned u64 arrays");
  if (temp_bytes < fs_histogram16_u64_temp_bytes(n))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes,
                fs_histogram16_u64_temp_bytes(n));
  const int grid = hist16_grid(n);
  char* t = (char*)temp;
  auto* spill = (unsigned long long*)t;
  auto* partials = (uint32_t*)(t + align_up(sizeof(uint64_t) * kHistBins));
  cudaError_t e = cudaMemsetAsync(spill, 0, sizeof(uint64_t) * kHistBins, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_histogram16_u64: memset");
  constexpr int smem = kHistWords * 4;
  if ((e = cudaFuncSetAttribute(k_digit_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
    return cuda_fail(e, "fs_histogram16_u64: smem attribute");
  k_digit_hist<<<grid, kThreads, smem, s>>>(keys, n, shift, (uint32_t)(nb - 1), partials, spill);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_histogram16_u64: k_digit_hist");
  if ((e = launch_merge_scan(partials, grid, spill, nullptr, kHistBins, hist, nb, 0, nullptr, nullptr, nullptr, s)) !=
      cudaSuccess)
    return cuda_fail(e, "fs_histogram16_u64: merge");
  return finish(s, "fs_histogram16_u64");
}

fs_status fs_select_bins_u64(const uint64_t* keys, uint64_t n, int shift, int width, const uint32_t* bins, int nb,
                             uint64_t* out, uint64_t cap, uint64_t* count, fs_stream_t stream) {
  FS_ENTRY();
  if (width < 1 || width > 16 || shift < 0 || shift + width > 64)
    return fail(FS_ERR_INVALID_ARGUMENT, "digit [shift %d, +%d) outside a u64 key or wider than 16 bits", shift,
                width);
  if (nb < 0 || nb > 64) return fail(FS_ERR_INVALID_ARGUMENT, "nb %d not in 0..64", nb);
  if (!count) return fail(FS_ERR_INVALID_ARGUMENT, "NULL count");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_select_bins_u64: memset");
  if (n == 0 || nb == 0) return finish(s, "fs_select_bins_u64");
  if (!keys || !bins || (cap && !out)) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  const uint64_t blocks = (n + 255) / 256;
  const unsigned grid = (unsigned)(blocks < (uint64_t)device_info().sm_count * 16 ? blocks
                                                                                   : (uint64_t)device_info().sm_count * 16);
  k_select_bins<<<grid, 256, 0, s>>>(keys, n, shift, (uint32_t)((1ull << width) - 1), bins, nb, out, cap,
                                     (unsigned long long*)count);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_select_bins_u64");
  return finish(s, "fs_select_bins_u64");
}

fs_status fs_digit_counts_sorted_u64(const uint64_t* sorted, uint64_t m, const uint64_t* prefixes, int np, int shift,
                                     int width, uint64_t* hist, fs_stream_t stream) {
  FS_ENTRY();
  if (width < 1 || width > 16 || shift < 0 || shift + width > 64)
    return fail(FS_ERR_INVALID_ARGUMENT, "digit [shift %d, +%d) outside a u64 key or wider than 16 bits", shift,
                width);
  if (np < 0) return fail(FS_ERR_INVALID_ARGUMENT, "np %d < 0", np);
  if (np == 0) return FS_OK;
  if (!prefixes || !hist || (m && !sorted)) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t total = (uint64_t)np << width;
  k_digit_counts_sorted<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(sorted, m, prefixes, np, shift, width, hist);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fs_digit_counts_sorted_u64");
  return finish(s, "fs_digit_counts_sorted_u64");
}

size_t fs_pair_exchange_temp_bytes(uint64_t n, int G) { return class_layout(n, G < 1 ? 1 : G).total; }

fs_status fs_pair_classes_u64(const uint64_t* keys, uint64_t n, const uint64_t* splitters, int G, uint64_t* class_tot,
                              void* temp, size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (G < 1 || G > kMaxG) return fail(FS_ERR_INVALID_ARGUMENT, "G %d not in 1..%d", G, kMaxG);
  if (!class_tot || !temp || (n && !keys) || (G > 1 && !splitters))
    return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  const ClassLayout L = class_layout(n, G);
  if (temp_bytes < L.total) return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, L.total);
  cudaStream_t s = (cudaStream_t)stream;
  char* t = (char*)temp;
  const int C = 2 * G - 1;
  const uint64_t ne = (uint64_t)C * (L.T ? L.T : 1);
  cudaError_t e;
  if (L.T == 0) {
    if ((e = cudaMemsetAsync(class_tot, 0, sizeof(uint64_t) * C, s)) != cudaSuccess)
      return cuda_fail(e, "fs_pair_classes_u64: memset");
    return finish(s, "fs_pair_classes_u64");
  }
  k_class_counts<<<(unsigned)L.T, kTileThreads, 0, s>>>(keys, n, splitters, G, (uint64_t*)(t + L.counts), L.T);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_pair_classes_u64: counts");
  fs_status st = fs_exclusive_scan_u64((uint64_t*)(t + L.counts), (uint64_t*)(t + L.off), (uint32_t)ne, t + L.stemp,
                                       L.stemp_bytes, stream);
  if (st != FS_OK) return st;
  k_class_totals<<<1, 64, 0, s>>>((uint64_t*)(t + L.off), L.T, C, class_tot);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_pair_classes_u64: totals");
  return finish(s, "fs_pair_classes_u64");
}

fs_status fs_pair_scatter_u64_u32(const uint64_t* keys, const uint32_t* vals, uint64_t n, const uint64_t* splitters,
                                  int G, const uint64_t* cuts_host, const uint64_t* bases_host,
                                  uint64_t* const* dest_keys_host, uint32_t* const* dest_vals_host, void* temp,
                                  size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (G < 1 || G > kMaxG) return fail(FS_ERR_INVALID_ARGUMENT, "G %d not in 1..%d", G, kMaxG);
  if (!cuts_host || !bases_host || !dest_keys_host || !dest_vals_host || !temp || (n && (!keys || !vals)) ||
      (G > 1 && !splitters))
    return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  const ClassLayout L = class_layout(n, G);
  if (temp_bytes < L.total) return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, L.total);
  if (cuts_host[0] != 0 || cuts_host[G] != n) return fail(FS_ERR_INVALID_ARGUMENT, "cuts must run from 0 to n");
  for (int d = 0; d < G; ++d) {
    if (cuts_host[d] > cuts_host[d + 1]) return fail(FS_ERR_INVALID_ARGUMENT, "cuts not ascending");
    if (cuts_host[d + 1] > cuts_host[d] && (!dest_keys_host[d] || !dest_vals_host[d]))
      return fail(FS_ERR_INVALID_ARGUMENT, "NULL destination for owner %d", d);
  }
  if (n == 0) return FS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  char* t = (char*)temp;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(t + L.cuts, cuts_host, sizeof(uint64_t) * (G + 1), cudaMemcpyHostToDevice, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(t + L.bases, bases_host, sizeof(uint64_t) * G, cudaMemcpyHostToDevice, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(t + L.dptr, dest_keys_host, sizeof(void*) * G, cudaMemcpyHostToDevice, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(t + L.dptr + sizeof(void*) * G, dest_vals_host, sizeof(void*) * G, cudaMemcpyHostToDevice,
                           s)) != cudaSuccess)
    return cuda_fail(e, "fs_pair_scatter_u64_u32: copy of the exchange plan");
  ScatterArgs a;
  a.keys = keys;
  a.vals = vals;
  a.n = n;
  a.T = L.T;
  a.splitters = splitters;
  a.G = G;
  a.off = (const uint64_t*)(t + L.off);
  a.cuts = (const uint64_t*)(t + L.cuts);
  a.bases = (const uint64_t*)(t + L.bases);
  a.dkeys = (uint64_t* const*)(t + L.dptr);
  a.dvals = (uint32_t* const*)(t + L.dptr + sizeof(void*) * G);
  k_class_scatter<<<(unsigned)L.T, kTileThreads, 0, s>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_pair_scatter_u64_u32");
  return finish(s, "fs_pair_scatter_u64_u32");
}

}  // extern "C"
