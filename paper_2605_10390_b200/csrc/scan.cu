// scan.cu — merge of the per-SM local histograms (stage 1b) fused with the
// single-pass decoupled-lookback exclusive scan over the bins (stage 2) (G2).
//
// Merge: C[v] = sum over CTAs of partial[cta][v] + spill[v] — the second step of
// the two-step High Precision Histogram Update (§III.A.1) and the
// Global Histogram Update (§III.B).
// Scan: P[v] = sum_{u<v} C[u], P[nbins] = N — Alg. 3 GetIndex(v) (PAPER.md:168-190,
// ledger 6) for every v at once; equally Alg. 5's running offset.
//
// B200 design: one CTA of 256 threads per tile of 256
// bins.  The partials (<= 148 x 128 KB, L2-resident) are read as 16-byte vectors
// by 8 row groups x 32 columns, so each warp reads 512 contiguous bytes per row.
// Tile order comes from an atomic ticket (never from blockIdx), so the lookback
// cannot wait on an unscheduled CTA.  Status words are 64-bit: 2-bit flag,
// 62-bit value (N up to 2^62), published with st.release.gpu and polled with
// ld.acquire.gpu.
#include "common.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 256;
static_assert(kScanTileBins == kThreads, "one bin per thread");
constexpr int kRowGroups = 8;                   // partial rows split across 8 warps
constexpr int kTileWords = kScanTileBins / 2;   // packed words per tile (128)
constexpr int kTileVec = kTileWords / 4;        // uint4 per tile row (32)

struct ScanSmem {
  uint32_t part[kRowGroups][kScanTileBins];
  unsigned long long warp_tot[kThreads / 32];
  unsigned long long exclusive;
  uint32_t tile;
};

template <bool kFromPartials>
__global__ void __launch_bounds__(kThreads)
    k_merge_scan(const uint32_t* __restrict__ partials, int parts, const unsigned long long* __restrict__ spill,
                 const uint64_t* __restrict__ hist_in, uint64_t nbins, uint64_t* __restrict__ hist_out,
                 uint64_t nbins_out, int accumulate, uint64_t* __restrict__ prefix,
                 unsigned long long* __restrict__ status, uint32_t* __restrict__ ticket) {
  __shared__ ScanSmem sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

  if (tid == 0) sm.tile = prefix ? atomicAdd(ticket, 1u) : blockIdx.x;
  __syncthreads();
  const uint64_t tile = sm.tile;
  const uint64_t bin = tile * kScanTileBins + tid;

  // ---- merge: this thread's bin count
  unsigned long long c = 0;
  if (kFromPartials) {
    const uint32_t col = tid & (kTileVec - 1), rg = tid >> 5;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint4* base = reinterpret_cast<const uint4*>(partials) + tile * kTileVec + col;
    constexpr uint64_t kRowVec = kHistWords / 4;
    int g = rg;
    for (; g + 3 * kRowGroups < parts; g += 4 * kRowGroups) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcg(base + (uint64_t)(g + u * kRowGroups) * kRowVec);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[0] += q[u].x & 0xFFFFu; acc[1] += q[u].x >> 16;
        acc[2] += q[u].y & 0xFFFFu; acc[3] += q[u].y >> 16;
        acc[4] += q[u].z & 0xFFFFu; acc[5] += q[u].z >> 16;
        acc[6] += q[u].w & 0xFFFFu; acc[7] += q[u].w >> 16;
      }
    }
    for (; g < parts; g += kRowGroups) {
      const uint4 q = __ldcg(base + (uint64_t)g * kRowVec);
      acc[0] += q.x & 0xFFFFu; acc[1] += q.x >> 16;
      acc[2] += q.y & 0xFFFFu; acc[3] += q.y >> 16;
      acc[4] += q.z & 0xFFFFu; acc[5] += q.z >> 16;
      acc[6] += q.w & 0xFFFFu; acc[7] += q.w >> 16;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.part[rg][col * 8 + j] = acc[j];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRowGroups; ++r) c += sm.part[r][tid];
    if (bin < nbins) c += spill[bin];
  } else {
    c = bin < nbins ? hist_in[bin] : 0ull;
  }
  if (hist_out && bin < nbins_out) hist_out[bin] = accumulate ? hist_out[bin] + c : c;
  if (!prefix) return;

  // ---- block exclusive scan of the 256 counts
  const unsigned long long inc = warp_inclusive_scan<unsigned long long>(c);
  if (lane == 31) sm.warp_tot[warp] = inc;
  __syncthreads();
  unsigned long long warp_off = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const unsigned long long t = sm.warp_tot[w];
    if (w < (int)warp) warp_off += t;
    agg += t;
  }
  const unsigned long long local_excl = warp_off + inc - c;

  // ---- decoupled lookback over earlier tiles
  if (warp == 0) {
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(&status[0], kFlagInclusive | agg);
    } else {
      if (lane == 0) st_relaxed_u64(&status[tile], kFlagAggregate | agg);
      int64_t base = (int64_t)tile - 1;
      while (true) {
        const int64_t idx = base - (int64_t)lane;
        unsigned long long s = idx >= 0 ? ld_relaxed_u64(&status[idx]) : kFlagInclusive;
        while (__any_sync(kFull, (s >> 62) == 0)) {
          if ((s >> 62) == 0) s = ld_relaxed_u64(&status[idx]);
        }
        const uint32_t incl_mask = __ballot_sync(kFull, (s >> 62) == 2);
        unsigned long long v = s & kValueMask;
        if (incl_mask) {
          const uint32_t first = __ffs(incl_mask) - 1;  // nearest inclusive predecessor
          if (lane > first) v = 0;
          excl += warp_sum(v);
          break;
        }
        excl += warp_sum(v);
        base -= 32;
      }
      if (lane == 0) st_relaxed_u64(&status[tile], kFlagInclusive | (excl + agg));
    }
    if (lane == 0) sm.exclusive = excl;
  }
  __syncthreads();
  const unsigned long long ex = sm.exclusive;
  if (bin < nbins) prefix[bin] = ex + local_excl;
  if (bin == nbins - 1) prefix[nbins] = ex + local_excl + c;
}

}  // namespace

cudaError_t launch_merge_scan(const uint32_t* partials, int parts, const unsigned long long* spill,
                              const uint64_t* hist_in, uint64_t nbins, uint64_t* hist_out, uint64_t nbins_out,
                              int accumulate, uint64_t* prefix, unsigned long long* status, uint32_t* ticket,
                              cudaStream_t s) {
  const uint64_t tiles = scan_tiles(nbins);
  if (tiles == 0) return cudaSuccess;
  if (hist_in)
    k_merge_scan<false><<<(unsigned)tiles, kThreads, 0, s>>>(partials, parts, spill, hist_in, nbins, hist_out,
                                                             nbins_out, accumulate, prefix, status, ticket);
  else
    k_merge_scan<true><<<(unsigned)tiles, kThreads, 0, s>>>(partials, parts, spill, hist_in, nbins, hist_out,
                                                            nbins_out, accumulate, prefix, status, ticket);
  return cudaGetLastError();
}

}  // namespace fs
