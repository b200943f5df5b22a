// expand16.cu — stage 3 of the u16 path: count-expansion (G3).
//
// What it computes: Alg. 5 ReconstructAll (§III.G.3) with
// t = p - l_n = 0 and l_b = 0 — the entries carry no bits, so bin b is emitted
// C[b] times in ascending b ("if C[b] = 0 continue").  Written as
// a function of output position j: out[j] = the v with P[v] <= j < P[v+1].
// Restricted to global positions [out_begin, out_end) so a rank of the
// multi-GPU path writes only its own range (SURVEY.md §8(e) Mode B).
//
// B200 design: HBM-write bound (2 B per key).
// Each CTA owns an output tile of kTile keys.  Warps 0 and 1 locate the first
// and last bin touching the tile with a 32-ary search of P in L2 (4 rounds for
// 65,536 bins); the tile's slice of P is staged in shared memory as 32-bit
// offsets relative to the tile; each thread then emits 8 keys per 16-byte
// streaming store (consecutive lanes -> consecutive 16 B), finding each run by
// binary search in the staged slice (one search per vector unless a run
// boundary falls inside it).  Unaligned head/tail keys are handled one per
// thread by CTA 0.
#include "common.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 256;
constexpr int kVecPerThread = 8;
constexpr uint64_t kTile = (uint64_t)kThreads * kVecPerThread * 8;  // 16,384 keys = 32 KB
constexpr int kSliceCap = 4096;                                    // staged P entries

// Largest v in [lo, hi) with P[v] <= o, given P[lo] <= o.  Whole warp participates.
FS_DEVINL uint64_t warp_last_le(const uint64_t* __restrict__ P, uint64_t lo, uint64_t hi, uint64_t o) {
  const uint32_t lane = lane_id();
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t idx = lo + lane * step;
    const bool ok = idx < hi && __ldcg(P + idx) <= o;
    const uint32_t m = __ballot_sync(kFull, ok);  // lane 0 always set
    const uint32_t L = 31 - __clz(m);
    lo = lo + L * step;
    const uint64_t nhi = lo + step;
    hi = nhi < hi ? nhi : hi;
  }
  const uint64_t idx = lo + lane;
  const bool ok = idx < hi && __ldcg(P + idx) <= o;
  const uint32_t m = __ballot_sync(kFull, ok);
  return lo + (31 - __clz(m));
}

// Thread-level binary search over global P: largest v in [lo, hi) with P[v] <= o.
FS_DEVINL uint64_t thread_last_le(const uint64_t* __restrict__ P, uint64_t lo, uint64_t hi, uint64_t o) {
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (__ldcg(P + mid) <= o) lo = mid; else hi = mid;
  }
  return lo;
}

// Largest j in [lo, hi) with rel[j] <= l, given rel[lo] <= l.
FS_DEVINL uint32_t smem_last_le(const uint32_t* rel, uint32_t lo, uint32_t hi, uint32_t l) {
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rel[mid] <= l) lo = mid; else hi = mid;
  }
  return lo;
}

struct ExpandSmem {
  uint64_t v_lo, v_hi;
  uint32_t rel[kSliceCap];
};

__global__ void __launch_bounds__(kThreads)
    k_expand16(const uint64_t* __restrict__ P, uint64_t nbins, uint64_t pos0, uint64_t nvec,
               uint16_t* __restrict__ out_body, uint64_t out_begin, uint64_t head, uint64_t tail_pos,
               uint64_t tail_n, uint16_t* __restrict__ out) {
  __shared__ ExpandSmem sm;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;

  // Unaligned head/tail keys (< 8 each): one per thread in CTA 0.
  if (blockIdx.x == 0 && tid < head + tail_n) {
    const uint64_t j = tid < head ? out_begin + tid : tail_pos + (tid - head);
    const uint64_t v = thread_last_le(P, 0, nbins, j);
    out[j - out_begin] = (uint16_t)v;
  }
  if (nvec == 0) return;

  const uint64_t vec0 = (uint64_t)blockIdx.x * (kTile / 8);
  const uint64_t vec_end = vec0 + kTile / 8 < nvec ? vec0 + kTile / 8 : nvec;
  const uint64_t o0 = pos0 + vec0 * 8;                 // first global position of the tile
  const uint32_t len = (uint32_t)((vec_end - vec0) * 8);
  if (warp == 0) {
    const uint64_t v = warp_last_le(P, 0, nbins, o0);
    if (lane_id() == 0) sm.v_lo = v;
  } else if (warp == 1) {
    const uint64_t v = warp_last_le(P, 0, nbins, o0 + len - 1);
    if (lane_id() == 0) sm.v_hi = v;
  }
  __syncthreads();
  const uint64_t v_lo = sm.v_lo, v_hi = sm.v_hi;
  const uint64_t m = v_hi - v_lo + 2;  // P[v_lo .. v_hi+1]
  uint4* dst = reinterpret_cast<uint4*>(out_body) + vec0;

  if (m <= (uint64_t)kSliceCap) {
    for (uint32_t j = tid; j < m; j += kThreads) {
      const uint64_t p = __ldcg(P + v_lo + j);
      sm.rel[j] = p <= o0 ? 0u : (p - o0 >= len ? len : (uint32_t)(p - o0));
    }
    __syncthreads();
    const uint32_t mm = (uint32_t)m;
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const uint32_t q = k * kThreads + tid;
      const uint32_t l = q * 8;
      if (l >= len) break;
      uint32_t j = smem_last_le(sm.rel, 0, mm - 1, l);
      uint32_t run_end = sm.rel[j + 1];
      uint32_t packed[4];
      if (l + 7 < run_end) {  // whole vector inside one run (common case)
        const uint32_t v = (uint32_t)(v_lo + j);
        const uint32_t pv = v | (v << 16);
        packed[0] = packed[1] = packed[2] = packed[3] = pv;
      } else {
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          uint32_t pair = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t pos = l + e + h;
            if (pos >= run_end) {
              j = smem_last_le(sm.rel, j + 1, mm - 1, pos);
              run_end = sm.rel[j + 1];
            }
            pair |= ((uint32_t)(v_lo + j) & 0xFFFFu) << (16 * h);
          }
          packed[e / 2] = pair;
        }
      }
      st_stream_v4(dst + q, make_uint4(packed[0], packed[1], packed[2], packed[3]));
    }
  } else {
    // Very sparse tile (more than kSliceCap bins): search P in L2 per position.
#pragma unroll 1
    for (int k = 0; k < kVecPerThread; ++k) {
      const uint32_t q = k * kThreads + tid;
      const uint32_t l = q * 8;
      if (l >= len) break;
      uint32_t packed[4] = {0, 0, 0, 0};
      uint64_t v = thread_last_le(P, v_lo, v_hi + 1, o0 + l);
      uint64_t run_end = __ldcg(P + v + 1);
      for (int e = 0; e < 8; ++e) {
        const uint64_t pos = o0 + l + e;
        if (pos >= run_end) {
          v = thread_last_le(P, v + 1, v_hi + 1, pos);
          run_end = __ldcg(P + v + 1);
        }
        packed[e / 2] |= ((uint32_t)v & 0xFFFFu) << (16 * (e & 1));
      }
      st_stream_v4(dst + q, make_uint4(packed[0], packed[1], packed[2], packed[3]));
    }
  }
}

}  // namespace

cudaError_t launch_expand16(const uint64_t* prefix, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                            uint16_t* out, cudaStream_t s) {
  const uint64_t n = out_end - out_begin;
  if (n == 0) return cudaSuccess;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(out);
  uint64_t head = ((16 - (addr & 15)) & 15) / 2;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 8;
  const uint64_t tail_n = n - head - nvec * 8;
  const uint64_t pos0 = out_begin + head;
  const uint64_t tail_pos = pos0 + nvec * 8;
  uint64_t grid = (nvec * 8 + kTile - 1) / kTile;
  if (grid == 0) grid = 1;
  k_expand16<<<(unsigned)grid, kThreads, 0, s>>>(prefix, nbins, pos0, nvec, out + head, out_begin, head, tail_pos,
                                                 tail_n, out);
  return cudaGetLastError();
}

}  // namespace fs
