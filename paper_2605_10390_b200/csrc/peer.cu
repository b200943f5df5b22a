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
// places — no local sort of the shard, no staging buffer, no all-to-all, no
// sort of what arrived (Mode A moves 4 + 2 + 2 + 4 B/key through HBM).  Lanes
// take consecutive j, so a warp's 32 stores are one contiguous 64 B run of a
// value (split only where a run crosses a rank boundary).
#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 32;  // positions per thread (strided by the warp width)

FS_DEVINL uint64_t range_begin(uint64_t d, uint64_t G, uint64_t N) {
  return (uint64_t)(((unsigned __int128)N * d) / G);
}

// tot[v] = sum_r C[r][v], cg[v] = C[g][v], below[v] = sum_{r<g} C[r][v].
__global__ void __launch_bounds__(kThreads)
    k_peer_counts(const uint64_t* __restrict__ C, int G, int g, uint64_t nbins, uint64_t* __restrict__ tot,
                  uint64_t* __restrict__ cg, uint64_t* __restrict__ below) {
  const uint64_t v = blockIdx.x * (uint64_t)kThreads + threadIdx.x;
  if (v >= nbins) return;
  uint64_t t = 0, b = 0;
  for (int r = 0; r < G; ++r) {
    const uint64_t c = C[(uint64_t)r * nbins + v];
    if (r < g) b += c;
    t += c;
  }
  tot[v] = t;
  cg[v] = C[(uint64_t)g * nbins + v];
  below[v] = b;
}

// Largest v < nbins with Pg[v] <= j (Pg[0] = 0 <= j).
FS_DEVINL uint64_t last_le(const uint64_t* Pg, uint64_t nbins, uint64_t j) {
  uint64_t lo = 0, hi = nbins;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(Pg + mid) <= j) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads)
    k_expand_to_peers(const uint64_t* __restrict__ P, const uint64_t* __restrict__ Pg,
                      const uint64_t* __restrict__ below, uint64_t nbins, int G, uint16_t* const* __restrict__ dest) {
  const uint64_t N = __ldg(P + nbins), ng = __ldg(Pg + nbins);
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (kThreads / 32);
  constexpr uint64_t kChunk = 32 * kPerThread;  // positions per warp chunk
  for (uint64_t w = (blockIdx.x * (uint64_t)kThreads + threadIdx.x) >> 5; w * kChunk < ng; w += nwarps) {
    uint64_t j = w * kChunk + lane;
    if (j >= ng) continue;  // (no warp collectives below)
    uint64_t v = last_le(Pg, nbins, j);
    uint64_t run_end = __ldg(Pg + v + 1);
    uint64_t run_pos = __ldg(P + v) + __ldg(below + v) - __ldg(Pg + v);  // global position = run_pos + j
    int d = (int)(((unsigned __int128)(run_pos + j) * G) / (N ? N : 1));
    if (d >= G) d = G - 1;
    for (int k = 0; k < kPerThread; ++k, j += 32) {
      if (j >= ng) break;
      while (j >= run_end) {  // the next non-empty value (runs are long: a short walk)
        ++v;
        run_end = __ldg(Pg + v + 1);
        run_pos = __ldg(P + v) + __ldg(below + v) - __ldg(Pg + v);
      }
      const uint64_t pos = run_pos + j;
      while (d + 1 < G && range_begin(d + 1, G, N) <= pos) ++d;
      while (d > 0 && range_begin(d, G, N) > pos) --d;
      dest[d][pos - range_begin(d, G, N)] = (uint16_t)v;
    }
  }
}

struct PeerLayout {
  size_t tot = 0, cg = 0, below = 0, P = 0, Pg = 0, scan1 = 0, scan2 = 0, dest = 0, zero_end = 0, total = 0;
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
  L.P = off;
  off = align_up(off + sizeof(uint64_t) * (nbins + 1));
  L.Pg = off;
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
  auto* P = (uint64_t*)(t + L.P);
  auto* Pg = (uint64_t*)(t + L.Pg);
  auto* s1 = (unsigned long long*)(t + L.scan1);
  auto* s2 = (unsigned long long*)(t + L.scan2);
  auto* dest = (uint16_t**)(t + L.dest);
  cudaError_t e;
  if ((e = cudaMemsetAsync(t, 0, L.zero_end, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(dest, dest_host, sizeof(void*) * (size_t)G, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  k_peer_counts<<<(unsigned)((nbins + kThreads - 1) / kThreads), kThreads, 0, s>>>(hist_all, G, g, nbins, tot, cg,
                                                                                 below);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint64_t st = scan_tiles(nbins);
  if ((e = launch_merge_scan(nullptr, 0, nullptr, tot, nbins, nullptr, 0, 0, P, s1, (uint32_t*)(s1 + st), s)) !=
      cudaSuccess)
    return e;
  if ((e = launch_merge_scan(nullptr, 0, nullptr, cg, nbins, nullptr, 0, 0, Pg, s2, (uint32_t*)(s2 + st), s)) !=
      cudaSuccess)
    return e;
  const unsigned grid = (unsigned)((uint64_t)device_info().sm_count * 8);  // warp-chunk loop covers any n
  k_expand_to_peers<<<grid, kThreads, 0, s>>>(P, Pg, below, nbins, G, dest);
  return cudaGetLastError();
}

}  // namespace fs
