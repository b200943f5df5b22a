// onesweep.cu — multi-digit precision scaling for u32/u64 keys and (u64, u32)
// pairs (config c5): stable LSD radix sort with 8-bit digits, one compressed
// histogram per digit (G4, G5; ledger 25).
//
// Paper passages: the "histogram, prefix sum and stable scatter phases" of radix
// sorting (§II); precision scaling; the index
// array I that "maps each sorted position to an arrival position"
// is what the values become when vals_in[i] = i, which requires stability.
//
// B200 design:
//  1. k_digit_hist: one read of the keys builds all ceil(key_bits/8) digit
//     histograms (256 bins each) in shared memory, merged into global u64.
//  2. k_digit_plan: exclusive scan per digit -> digit_base; a digit whose
//     histogram has a single non-empty bin is skipped; the ping-pong parity of
//     every executed pass is fixed on the device so the last pass lands in the
//     caller's output (no host synchronisation).
//  3. k_onesweep (per digit): tiles of 3072 keys (256 threads x 12 items, 4
//     CTAs per SM) taken in order from an atomic ticket; warp-level ranking with
//     an 8-ballot multisplit (input order preserved: item-major, lane-minor
//     within a warp chunk, warps in order; match.any measured ~10x slower);
//     per-tile digit counts published to a 64-bit status word per (tile, digit)
//     [flag:2 | pass tag:6 | value:56] with relaxed stores; decoupled lookback,
//     one thread per digit, 8 predecessors fetched per round; keys (and values)
//     reordered through shared memory so each digit's run is written with
//     consecutive addresses.
#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 12;
constexpr int kTileKeys = kThreads * kItems;  // 3072
static_assert(kThreads == kRadix, "one thread per digit in the lookback");

constexpr unsigned long long kStFlagAgg = 1ull << 62;
constexpr unsigned long long kStFlagInc = 2ull << 62;
constexpr int kTagShift = 56;
constexpr unsigned long long kStValue = (1ull << kTagShift) - 1;

struct Plan {
  uint64_t base[kMaxPasses][kRadix];  // exclusive digit offsets
  uint32_t skip[kMaxPasses];
  uint32_t exec_index[kMaxPasses];    // 1-based index among executed passes
  uint32_t executed;                  // E
};

template <typename K>
FS_DEVINL uint32_t digit_of(K key, int shift) {
  return (uint32_t)(key >> shift) & (kRadix - 1);
}

// ---------------------------------------------------------------- histogram
template <typename K>
__global__ void __launch_bounds__(512)
    k_digit_hist(const K* __restrict__ keys, uint64_t n, int passes, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t sh[kMaxPasses * kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = __ldcs(keys + i);
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < passes) atomicAdd(&sh[p * kRadix + digit_of(k, p * kRadixBits)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

__global__ void __launch_bounds__(kRadix)
    k_digit_plan(const unsigned long long* __restrict__ hist, uint64_t n, int passes, Plan* __restrict__ plan) {
  __shared__ uint32_t skip_sh[kMaxPasses];
  __shared__ unsigned long long wsum[kRadix / 32];
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  if (d < kMaxPasses) skip_sh[d] = 0;
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    const unsigned long long c = hist[p * kRadix + d];
    if (c == n) skip_sh[p] = 1;  // every key has this digit: the pass is the identity
    const unsigned long long inc = warp_inclusive_scan<unsigned long long>(c);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned long long off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    plan->base[p][d] = off + inc - c;
    __syncthreads();
  }
  if (d == 0) {
    uint32_t e = 0;
    for (int p = 0; p < kMaxPasses; ++p) {
      const uint32_t s = p < passes ? skip_sh[p] : 1u;
      plan->skip[p] = s;
      if (!s) ++e;
      plan->exec_index[p] = s ? 0u : e;
    }
    plan->executed = e;
  }
}

// ---------------------------------------------------------------- scatter pass
template <typename K, bool kHasValues>
struct PassSmem {
  K stage_k[kTileKeys];
  uint32_t stage_v[kHasValues ? kTileKeys : 1];
  uint32_t whist[kWarps][kRadix];      // per-warp counts, then per-warp exclusive offsets
  uint32_t digit_start[kRadix];        // tile-local exclusive scan over digits
  unsigned long long gofs[kRadix];     // global offset - digit_start
  uint32_t wsum[kWarps];
  uint32_t tile;
};

template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kThreads, 4)
    k_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kX,
               uint32_t* __restrict__ vX, K* __restrict__ kY, uint32_t* __restrict__ vY, uint64_t n, int pass,
               const Plan* __restrict__ plan, unsigned long long* __restrict__ status, uint32_t* __restrict__ ticket) {
  if (plan->skip[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<PassSmem<K, kHasValues>*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const int shift = pass * kRadixBits;
  const unsigned long long tag = (unsigned long long)(pass + 1) << kTagShift;

  // Buffers of this pass (ping-pong fixed on the device, see k_digit_plan).
  const uint32_t E = plan->executed, e = plan->exec_index[pass];
  const bool dst_is_x = ((E - e) & 1u) == 0;
  const K* src_k = e == 1 ? kin : (dst_is_x ? kY : kX);
  const uint32_t* src_v = e == 1 ? vin : (dst_is_x ? vY : vX);
  K* dst_k = dst_is_x ? kX : kY;
  uint32_t* dst_v = dst_is_x ? vX : vY;

  if (tid == 0) sm.tile = atomicAdd(ticket, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&sm.whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = sm.tile;
  const uint64_t tile0 = tile * kTileKeys;
  const uint64_t chunk0 = tile0 + (uint64_t)warp * 32 * kItems;

  // ---- load (warp-striped: item i of lane l is element chunk0 + 32 i + l)
  K key[kItems];
  uint32_t val[kHasValues ? kItems : 1];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = chunk0 + 32 * i + lane;
    key[i] = idx < n ? __ldcs(src_k + idx) : K(0);
    if (kHasValues) val[i] = idx < n ? __ldcs(src_v + idx) : 0u;
  }

  // ---- warp-level stable ranking
  uint32_t rank[kItems];
  uint32_t* wh = sm.whist[warp];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = chunk0 + 32 * i + lane < n;
    const uint32_t d = digit_of(key[i], shift);
    // lanes holding the same digit: 8 ballots (match.any is far slower on sm_100a)
    uint32_t peers = __ballot_sync(kFull, valid);
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t vote = __ballot_sync(kFull, bit);
      peers &= bit ? vote : ~vote;
    }
    const uint32_t leader = 31 - __clz(peers);
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = wh[d];
      wh[d] = old + __popc(peers);
    }
    old = __shfl_sync(kFull, old, leader);
    rank[i] = old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();

  // ---- tile digit counts, per-warp offsets, tile-local digit starts (thread = digit)
  const uint32_t d = tid;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = sm.whist[w][d];
    sm.whist[w][d] = cnt;
    cnt += c;
  }
  const uint32_t inc = warp_inclusive_scan<uint32_t>(cnt);
  if (lane == 31) sm.wsum[warp] = inc;

  // publish this tile's count for digit d, then look back over earlier tiles
  unsigned long long* st = status + tile * kRadix + d;
  unsigned long long excl = 0;
  if (tile == 0) {
    st_relaxed_u64(st, kStFlagInc | tag | cnt);
  } else {
    st_relaxed_u64(st, kStFlagAgg | tag | cnt);
    // Look back kLook predecessors per round: their status loads are independent,
    // so a round costs one L2 round trip instead of kLook.  Walk them in order
    // (nearest first), summing aggregates until an inclusive prefix.
    constexpr int kLook = 8;
    int64_t t = (int64_t)tile - 1;
    bool done = false;
    while (!done) {
      unsigned long long sv[kLook];
#pragma unroll
      for (int j = 0; j < kLook; ++j)
        sv[j] = t - j >= 0 ? ld_relaxed_u64(status + (uint64_t)(t - j) * kRadix + d) : (kStFlagInc | tag);
#pragma unroll
      for (int j = 0; j < kLook; ++j) {
        if (done) break;
        unsigned long long s = sv[j];
        while ((s & (0x3Full << kTagShift)) != tag || (s >> 62) == 0)  // not yet published: wait for it
          s = ld_relaxed_u64(status + (uint64_t)(t - j) * kRadix + d);
        excl += s & kStValue;
        done = (s >> 62) == 2;
      }
      t -= kLook;
    }
    st_relaxed_u64(st, kStFlagInc | tag | (excl + cnt));
  }
  __syncthreads();
  uint32_t woff = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w)
    if (w < (int)warp) woff += sm.wsum[w];
  const uint32_t dstart = woff + inc - cnt;
  sm.digit_start[d] = dstart;
  sm.gofs[d] = plan->base[pass][d] + excl - dstart;
  __syncthreads();

  // ---- reorder through shared memory
  const uint64_t rem = n - tile0;
  const uint32_t valid_count = rem < (uint64_t)kTileKeys ? (uint32_t)rem : (uint32_t)kTileKeys;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (chunk0 + 32 * i + lane < n) {
      const uint32_t dd = digit_of(key[i], shift);
      const uint32_t pos = sm.digit_start[dd] + wh[dd] + rank[i];
      sm.stage_k[pos] = key[i];
      if (kHasValues) sm.stage_v[pos] = val[i];
    }
  }
  __syncthreads();

  // ---- scatter: consecutive positions of one digit go to consecutive addresses
  for (uint32_t j = tid; j < valid_count; j += kThreads) {
    const K k = sm.stage_k[j];
    const uint64_t dst = sm.gofs[digit_of(k, shift)] + j;
    dst_k[dst] = k;
    if (kHasValues) dst_v[dst] = sm.stage_v[j];
  }
}

// If every pass was skipped (all keys share every digit), the output is the input.
template <typename K, bool kHasValues>
__global__ void k_copy_if_identity(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
                                   uint32_t* __restrict__ vout, uint64_t n, const Plan* __restrict__ plan) {
  if (plan->executed != 0) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    kout[i] = kin[i];
    if (kHasValues) vout[i] = vin[i];
  }
}

struct OnesweepLayout {
  size_t alt_k = 0, alt_v = 0, hist = 0, tickets = 0, status = 0, zero_end = 0, plan = 0, total = 0;
  uint64_t tiles = 0;
};

OnesweepLayout layout(uint64_t n, int key_bytes, int key_bits, bool has_values) {
  OnesweepLayout L;
  const int width = key_bytes * 8;
  if (key_bits <= 0 || key_bits > width) key_bits = width;
  const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
  L.tiles = (n + kTileKeys - 1) / kTileKeys;
  size_t off = 0;
  L.alt_k = off;
  off = align_up(off + (size_t)n * key_bytes);
  L.alt_v = off;
  if (has_values) off = align_up(off + (size_t)n * 4);
  L.hist = off;  // zeroed region starts here
  off = align_up(off + sizeof(unsigned long long) * kMaxPasses * kRadix);
  L.tickets = off;
  off = align_up(off + sizeof(uint32_t) * kMaxPasses);
  L.status = off;
  off = align_up(off + sizeof(unsigned long long) * kRadix * L.tiles * (passes > 0 ? 1 : 0));
  L.zero_end = off;
  L.plan = off;
  off = align_up(off + sizeof(Plan));
  L.total = off;
  return L;
}

template <typename K, bool kHasValues>
cudaError_t run(const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, uint64_t n, int key_bits, void* temp,
                cudaStream_t s) {
  const OnesweepLayout L = layout(n, sizeof(K), key_bits, kHasValues);
  const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
  char* t = (char*)temp;
  K* alt_k = (K*)(t + L.alt_k);
  uint32_t* alt_v = kHasValues ? (uint32_t*)(t + L.alt_v) : nullptr;
  auto* hist = (unsigned long long*)(t + L.hist);
  auto* tickets = (uint32_t*)(t + L.tickets);
  auto* status = (unsigned long long*)(t + L.status);
  auto* plan = (Plan*)(t + L.plan);

  phase_event(0, s);
  cudaError_t e = cudaMemsetAsync(t + L.hist, 0, L.zero_end - L.hist, s);
  if (e != cudaSuccess) return e;
  const int sms = device_info().sm_count;
  uint64_t hgrid = (n + 511) / 512;
  if (hgrid > (uint64_t)sms * 4) hgrid = (uint64_t)sms * 4;
  k_digit_hist<K><<<(unsigned)hgrid, 512, 0, s>>>(kin, n, passes, hist);
  k_digit_plan<<<1, kRadix, 0, s>>>(hist, n, passes, plan);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  phase_event(1, s);

  constexpr int smem = (int)sizeof(PassSmem<K, kHasValues>);
  e = cudaFuncSetAttribute(k_onesweep<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  for (int p = 0; p < passes; ++p) {
    k_onesweep<K, kHasValues><<<(unsigned)L.tiles, kThreads, smem, s>>>(
        kin, vin, kout, vout, alt_k, alt_v, n, p, plan, status + (size_t)0, tickets + p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    phase_event(2 + p, s);
  }
  k_copy_if_identity<K, kHasValues><<<(unsigned)(sms * 4), 256, 0, s>>>(kin, vin, kout, vout, n, plan);
  phase_event(2 + passes, s);
  return cudaGetLastError();
}

}  // namespace

size_t onesweep_temp_bytes(uint64_t n, int key_bytes, int key_bits, bool has_values) {
  return layout(n, key_bytes, key_bits, has_values).total;
}

cudaError_t onesweep_sort(const void* keys_in, const uint32_t* vals_in, void* keys_out, uint32_t* vals_out,
                          uint64_t n, int key_bytes, int key_bits, void* temp, size_t temp_bytes, cudaStream_t s) {
  (void)temp_bytes;
  if (key_bytes == 4)
    return run<uint32_t, false>((const uint32_t*)keys_in, nullptr, (uint32_t*)keys_out, nullptr, n, key_bits, temp, s);
  if (vals_in)
    return run<uint64_t, true>((const uint64_t*)keys_in, vals_in, (uint64_t*)keys_out, vals_out, n, key_bits, temp,
                               s);
  return run<uint64_t, false>((const uint64_t*)keys_in, nullptr, (uint64_t*)keys_out, nullptr, n, key_bits, temp, s);
}

}  // namespace fs
