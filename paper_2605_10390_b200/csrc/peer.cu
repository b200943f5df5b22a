// peer.cu — fused expand-to-peer exchange of the multi-GPU keys-only path
// (§8(e) Mode A without the staging passes).
//
// What it computes: with the gathered per-rank histograms C_r (the Global
// Histogram Update of PAPER.md:91-92 taken across GPUs), P = exclusive scan of
// sum_r C_r (Alg. 3 GetIndex for every value), rank g's keys of value v occupy
// the global sorted positions [P[v] + S_<g[v], P[v] + S_<=g[v]) — lower rank
// first (ledger 13) — and rank d owns positions
// [floor(dN/G), floor((d+1)N/G)) (ledger 23).  Rank g's j-th key in its own
// sorted order (value v, Pg[v] <= j < Pg[v+1], Pg = local exclusive scan) is
// therefore written to global position P[v] + S_<g[v] + (j - Pg[v]), i.e. into
// the output buffer of the rank that owns that position: Alg. 5's count
// expansion done by the producer straight into the
// consumer's memory.
//
// B200 design: the destination buffers are peer mappings (CUDA IPC over
// NVLink/NVSwitch); each rank streams its n_g keys (2 B each) to their final
// places -- no local sort of the shard, no staging buffer, no all-to-all, no
// sort of what arrived (Mode A moves 4 + 2 + 2 + 4 B/key through HBM).  Rank g's
// keys of value v form ONE contiguous run of the global output,
// [P[v] + S_<g[v], P[v] + S_<=g[v]); so the exchange is a set of fills.  Every run
// is cut into chunks of kChunk keys (and at the owners' range boundaries); a warp
// fills a chunk with 16-byte stores (v replicated eight times; lanes take
// consecutive 16 B, so a warp instruction is one 512 B burst over NVLink), the
// unaligned head and tail of the chunk with 2-byte stores.  The chunk list is the
// exclusive scan of ceil(C_g[v] / kChunk) (decoupled-lookback scan, scan.cu).
#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 256;
constexpr uint64_t kChunk = 8192;  // keys per chunk (16 KB: 32 store instructions per warp)

FS_DEVINL uint64_t range_begin(uint64_t d, uint64_t G, uint64_t N) {
  return (uint64_t)(((unsigned __int128)N * d) / G);
}

// tot[v] = sum_r C[r][v], cg[v] = C[g][v], below[v] = sum_{r<g} C[r][v],
// nch[v] = chunks of rank g's run of v.
__global__ void __launch_bounds__(kThreads)
    k_peer_counts(const uint64_t* __restrict__ C, int G, int g, uint64_t nbins, uint64_t* __restrict__ tot,
                  uint64_t* __restrict__ cg, uint64_t* __restrict__ below, uint64_t* __restrict__ nch) {
  const uint64_t v = blockIdx.x * (uint64_t)kThreads + threadIdx.x;
  if (v >= nbins) return;
  uint64_t t = 0, b = 0;
  for (int r = 0; r < G; ++r) {
    const uint64_t c = C[(uint64_t)r * nbins + v];
    if (r < g) b += c;
    t += c;
  }
  const uint64_t c = C[(uint64_t)g * nbins + v];
  tot[v] = t;
  cg[v] = c;
  below[v] = b;
  nch[v] = (c + kChunk - 1) / kChunk;
}

// Largest v < nbins with CB[v] <= c (CB[0] = 0 <= c).
FS_DEVINL uint64_t last_le(const uint64_t* CB, uint64_t nbins, uint64_t c) {
  uint64_t lo = 0, hi = nbins;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldcg(CB + mid) <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// dst[0 .. m) = v (one warp): 2-byte stores up to 16-byte alignment, 16-byte
// stores, 2-byte stores for the tail.
FS_DEVINL void warp_fill(uint16_t* dst, uint64_t m, uint16_t v, uint32_t lane) {
  const uint64_t head = min(m, (uint64_t)(((16 - ((uintptr_t)dst & 15)) & 15) >> 1));
  if (lane < head) dst[lane] = v;
  const uint64_t nvec = (m - head) >> 3;
  uint4* body = reinterpret_cast<uint4*>(dst + head);
  const uint32_t w = (uint32_t)v | ((uint32_t)v << 16);
  const uint4 q = make_uint4(w, w, w, w);
  for (uint64_t i = lane; i < nvec; i += 32) st_stream_v4(body + i, q);
  const uint64_t t0 = head + (nvec << 3);
  if (t0 + lane < m) dst[t0 + lane] = v;
}

__global__ void __launch_bounds__(kThreads)
    k_expand_to_peers(const uint64_t* __restrict__ P, const uint64_t* __restrict__ cg,
                      const uint64_t* __restrict__ below, const uint64_t* __restrict__ CB, uint64_t nbins, int G,
                      uint16_t* const* __restrict__ dest) {
  const uint64_t N = __ldcg(P + nbins), K = __ldcg(CB + nbins);
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (kThreads / 32);
  for (uint64_t c = (blockIdx.x * (uint64_t)kThreads + threadIdx.x) >> 5; c < K; c += nwarps) {
    const uint64_t v = last_le(CB, nbins, c);
    const uint64_t i0 = (c - __ldcg(CB + v)) * kChunk;
    const uint64_t len = min(kChunk, __ldcg(cg + v) - i0);
    uint64_t q0 = __ldcg(P + v) + __ldcg(below + v) + i0;  // first global position of the chunk
    const uint64_t q1 = q0 + len;
    int d = (int)(((unsigned __int128)q0 * G) / (N ? N : 1));
    if (d >= G) d = G - 1;
    while (d + 1 < G && range_begin(d + 1, G, N) <= q0) ++d;
    while (d > 0 && range_begin(d, G, N) > q0) --d;
    while (q0 < q1) {  // the pieces of the chunk in consecutive owners' ranges
      const uint64_t rb = range_begin(d, G, N), re = range_begin(d + 1, G, N);
      const uint64_t e = q1 < re ? q1 : re;
      warp_fill(dest[d] + (q0 - rb), e - q0, (uint16_t)v, lane);
      q0 = e;
      ++d;
    }
  }
}

struct PeerLayout {
  size_t tot = 0, cg = 0, below = 0, nch = 0, P = 0, CB = 0, scan1 = 0, scan2 = 0, dest = 0, zero_end = 0,
         total = 0;
};

PeerLayout peer_layout(uint64_t nbins, int G) {
  PeerLayout L;
  size_t off = 0;
  L.scan1 = off;  // scan status + ticket (zeroed)
  off = align_up(off + sizeof(uint64_t) * (scan_tiles(nbins) + 1));
  L.scan2 = off;
  off = align_up(off + sizeof(uint64_t) * (scan_tiles(nbins) + 1));
  L.zero_end = off;
  L.tot = off;
  off = align_up(off + sizeof(uint64_t) * nbins);
  L.cg = off;
  off = align_up(off + sizeof(uint64_t) * nbins);
  L.below = off;
  off = align_up(off + sizeof(uint64_t) * nbins);
  L.nch = off;
  off = align_up(off + sizeof(uint64_t) * nbins);
  L.P = off;
  off = align_up(off + sizeof(uint64_t) * (nbins + 1));
  L.CB = off;
  off = align_up(off + sizeof(uint64_t) * (nbins + 1));
  L.dest = off;
  off = align_up(off + sizeof(void*) * (size_t)G);
  L.total = off;
  return L;
}

}  // namespace

size_t expand_to_peers_temp_bytes(uint64_t nbins, int G) { return peer_layout(nbins, G).total; }

cudaError_t launch_expand_to_peers(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint16_t* const* dest_host,
                                   void* temp, cudaStream_t s) {
  const PeerLayout L = peer_layout(nbins, G);
  char* t = (char*)temp;
  auto* tot = (uint64_t*)(t + L.tot);
  auto* cg = (uint64_t*)(t + L.cg);
  auto* below = (uint64_t*)(t + L.below);
  auto* nch = (uint64_t*)(t + L.nch);
  auto* P = (uint64_t*)(t + L.P);
  auto* CB = (uint64_t*)(t + L.CB);
  auto* s1 = (unsigned long long*)(t + L.scan1);
  auto* s2 = (unsigned long long*)(t + L.scan2);
  auto* dest = (uint16_t**)(t + L.dest);
  cudaError_t e;
  if ((e = cudaMemsetAsync(t, 0, L.zero_end, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(dest, dest_host, sizeof(void*) * (size_t)G, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  k_peer_counts<<<(unsigned)((nbins + kThreads - 1) / kThreads), kThreads, 0, s>>>(hist_all, G, g, nbins, tot, cg,
                                                                                 below, nch);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint64_t st = scan_tiles(nbins);
  if ((e = launch_merge_scan(nullptr, 0, nullptr, tot, nbins, nullptr, 0, 0, P, s1, (uint32_t*)(s1 + st), s)) !=
      cudaSuccess)
    return e;
  if ((e = launch_merge_scan(nullptr, 0, nullptr, nch, nbins, nullptr, 0, 0, CB, s2, (uint32_t*)(s2 + st), s)) !=
      cudaSuccess)
    return e;
  const unsigned grid = (unsigned)((uint64_t)device_info().sm_count * 8);  // the warp loop covers any chunk count
  k_expand_to_peers<<<grid, kThreads, 0, s>>>(P, cg, below, CB, nbins, G, dest);
  return cudaGetLastError();
}

}  // namespace fs
