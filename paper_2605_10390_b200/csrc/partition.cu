// partition.cu — the exchange plan of the multi-GPU payload path (G7, Mode A).
//
// Exact, sampling-free splitters (ledger 13, 23): rank d owns
// global sorted positions [floor(d*N/G), floor((d+1)*N/G)).  After the gathered
// per-rank histograms C_r (the global histogram merge of PAPER.md:92 across
// GPUs), rank g's keys of value v occupy positions [P[v] + S_<g[v], P[v] +
// S_<=g[v]) where P is the exclusive scan of sum_r C_r (Alg. 3 GetIndex) and
// lower ranks come first (SPEC.md:309 tie-break).  send[d] counts how many of
// those positions fall in rank d's range, which is also the length of the
// slice of g's locally sorted keys that goes to d.
//
// One CTA of 1024 threads; each thread owns 64 consecutive bins (two passes:
// totals for a block scan, then overlap accumulation in shared memory).
#include "common.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 1024;
constexpr int kMaxRanks = 1024;

FS_DEVINL uint64_t range_begin(uint64_t d, uint64_t G, uint64_t N) {
  return (uint64_t)(((unsigned __int128)N * d) / G);
}

__global__ void __launch_bounds__(kThreads)
    k_send_counts(const uint64_t* __restrict__ C, int G, int g, uint64_t nbins, uint64_t* __restrict__ send) {
  __shared__ unsigned long long acc[kMaxRanks];
  __shared__ unsigned long long warp_tot[kThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (int d = tid; d < G; d += kThreads) acc[d] = 0;

  const uint64_t per = (nbins + kThreads - 1) / kThreads;
  const uint64_t v0 = tid * per < nbins ? tid * per : nbins;
  const uint64_t v1 = v0 + per < nbins ? v0 + per : nbins;

  unsigned long long mine = 0;
  for (uint64_t v = v0; v < v1; ++v)
    for (int r = 0; r < G; ++r) mine += C[(uint64_t)r * nbins + v];

  const unsigned long long inc = warp_inclusive_scan<unsigned long long>(mine);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  unsigned long long base = 0, N = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < (int)warp) base += warp_tot[w];
    N += warp_tot[w];
  }
  base += inc - mine;
  __syncthreads();

  unsigned long long Pv = base;
  for (uint64_t v = v0; v < v1; ++v) {
    unsigned long long below = 0, tot = 0;
    for (int r = 0; r < G; ++r) {
      const uint64_t c = C[(uint64_t)r * nbins + v];
      if (r < g) below += c;
      tot += c;
    }
    const uint64_t cg = C[(uint64_t)g * nbins + v];
    const uint64_t lo = Pv + below, hi = lo + cg;
    if (cg) {
      // first rank whose range ends after lo
      int d_lo = 0, d_hi = G - 1;
      while (d_lo < d_hi) {
        const int mid = (d_lo + d_hi) >> 1;
        if (range_begin(mid + 1, G, N) > lo) d_hi = mid; else d_lo = mid + 1;
      }
      for (int d = d_lo; d < G; ++d) {
        const uint64_t b0 = range_begin(d, G, N), b1 = range_begin(d + 1, G, N);
        if (b0 >= hi) break;
        const uint64_t a = lo > b0 ? lo : b0, b = hi < b1 ? hi : b1;
        if (b > a) atomicAdd(&acc[d], (unsigned long long)(b - a));
      }
    }
    Pv += tot;
  }
  __syncthreads();
  for (int d = tid; d < G; d += kThreads) send[d] = acc[d];
}

}  // namespace

cudaError_t launch_send_counts(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint64_t* send,
                               cudaStream_t s) {
  k_send_counts<<<1, kThreads, 0, s>>>(hist_all, G, g, nbins, send);
  return cudaGetLastError();
}

}  // namespace fs

// ---------------------------------------------------------------------------
// Exact splitters of the distributed pair sort (SURVEY.md §8(e) Mode A for
// pairs): the rank of a probe key in a rank's locally sorted keys.
// out[i] = #{j : sorted[j] < q[i]} (upper = 0) or #{j : sorted[j] <= q[i]}
// (upper = 1): one thread per probe, binary search over the sorted shard.
namespace fs {
namespace {
__global__ void __launch_bounds__(256) k_bound_u64(const uint64_t* __restrict__ sorted, uint64_t n,
                                                   const uint64_t* __restrict__ q, uint64_t nq, int upper,
                                                   uint64_t* __restrict__ out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const uint64_t x = q[i];
  uint64_t lo = 0, hi = n;  // first index whose key is >= x (lower) / > x (upper)
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    const uint64_t k = __ldg(sorted + mid);
    if (upper ? (k <= x) : (k < x)) lo = mid + 1; else hi = mid;
  }
  out[i] = lo;
}
}  // namespace

cudaError_t launch_bound_u64(const uint64_t* sorted, uint64_t n, const uint64_t* q, uint64_t nq, int upper,
                             uint64_t* out, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  k_bound_u64<<<(unsigned)((nq + 255) / 256), 256, 0, s>>>(sorted, n, q, nq, upper, out);
  return cudaGetLastError();
}
}  // namespace fs
