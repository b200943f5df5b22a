// wide.cu — multi-digit precision scaling for u32/u64 keys and (u64, u32) pairs
// (config c5).
//
// Two bit-identical schemes (the stable sort is unique, ledger 28):
//
// (1) Trie-binned MSD (default for n >= FS_MSD_MIN_N = FS_SMALL_SORT_MSD_MAX + 1
//     = 8,961 keys when key_bits >= 32; below, and up to kSmallSortMax = 16,384
//     keys when key_bits < 32, the one-CTA LSD k_small_sort).  The paper's
//     high-precision path (§III.G.3, Alg. 5) bins the keys by
//     the top levels of the compressed trie and then sorts each bin by its
//     remaining bits (per-bin radix), with the index array I
//     carried along:
//       a. k_top16_hist: one read of the keys builds the leaf level of a
//          16-level compressed trie over the key's top 16 bits (u16 counters
//          packed two per word in shared memory; overflow
//          spill as in hist16.cu), merged and scanned into P16 (scan.cu).  The
//          level-8 counters of that trie (sums of 256 leaves) are the bucket
//          bounds of the first MSD digit, the leaves those of the second — no
//          second histogram is needed.
//       b. k_scatter mode 1: stable scatter by bits [kb-8, kb) into the
//          temporary buffer; mode 2: stable scatter by bits [kb-16, kb-8)
//          within each of the 256 first-level segments, into the output.
//       c. every 16-bit bin is sorted in shared memory by its remaining kb-16
//          bits, stably, in place: k_local_sort (512 threads, <= kLocalCap
//          keys), k_local_mid (256 threads, <= kMidCap keys, four per SM),
//          k_tiny_bins (one warp per bin of <= kTinyMax keys); k_bin_lists
//          builds their lists.
//       d. k_heavy (wide_heavy.cuh): bins above kLocalCap recurse on the next
//          8-bit digits until every piece fits; k_heavy_items sorts the pieces.
//          k_heavy also runs level 2 for first-level buckets too large for the
//          interleaved lookback of (b).
//       e. a common key prefix moves the 16 bits' window below it
//          (k_binbits / k_keybits, then k_top16_hist again).
//     Traffic: 8 (u64 key read) + 3 x 24 = 80 B/pair for c5 (vs 200 for LSD-8);
//     each recursion level adds 8 + 24 B per pair of the oversize bins.
// (2) Stable LSD with 8-bit digits (small n, fewer than 32 varying key bits):
//     one read builds all digit histograms (k_digit_hist), k_digit_plan scans
//     them and skips single-bin digits, then one k_scatter (mode 0) per digit;
//     n <= FS_SMALL_SORT_MSD_MAX (<= kSmallSortMax for key_bits < 32): the same
//     LSD in one CTA's shared memory (k_small_sort).
//
// Choice: the host picks by n and key_bits; then the MSD path is taken unless
// one 16-bit bin holds every key after the window moved (then the MSD levels
// would move everything for nothing and LSD skips the uniform digits) —
// decided on the device, so nothing synchronises with the host; the kernels of
// the path not taken return at once.
//
// k_scatter (the "histogram, prefix sum and stable scatter phases"):
// persistent CTAs (2 per SM for pairs) take 4,096-key tiles in order from an
// atomic ticket; the next tile's keys and values are prefetched into shared
// memory with bulk copies (TMA) completing on an mbarrier while the current tile
// is ranked (8-ballot warp multisplit, stable: item-major, lane-minor, warps in
// order), its digit counts published to a 64-bit status word per (tile, digit)
// [flag:2 | pass tag:6 | count:56], reordered through shared memory, offset by a
// decoupled lookback (one thread per digit, 8 predecessors per round, never
// crossing a segment start) and written with consecutive addresses per digit.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "internal.cuh"
#include "kernels.cuh"
#include "tma.cuh"

#ifdef FS_SCATTER_STATS  // scripts/microbench/scatter_stats.cu: lookback behaviour per mode
__device__ unsigned long long g_scatter_stats[3][4];  // [mode][lookbacks, rounds, polls, inc_at_first]
__device__ unsigned long long g_scatter_phase[3][8];  // [mode][phase] clock cycles summed over CTAs (thread 0)
__device__ unsigned long long g_local_phase[8];       // local sort phases (thread 0 of each CTA)
#define FS_LPH(i)                                                        \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      const long long now_ = clock64();                                  \
      atomicAdd(&g_local_phase[i], (unsigned long long)(now_ - lph_t0)); \
      lph_t0 = now_;                                                     \
    }                                                                    \
  } while (0)
#define FS_PH(i)                                                            \
  do {                                                                     \
    if (tid == 0) {                                                        \
      const long long now_ = clock64();                                    \
      atomicAdd(&g_scatter_phase[a.mode][i], (unsigned long long)(now_ - ph_t0)); \
      ph_t0 = now_;                                                        \
    }                                                                      \
  } while (0)
#else
#define FS_PH(i) \
  do {           \
  } while (0)
#define FS_LPH(i) \
  do {            \
  } while (0)
#endif

namespace fs {
namespace {

#ifndef FS_WIDE_PDL
#define FS_WIDE_PDL 1
#endif
// Programmatic dependent launch between the path's kernels: a kernel launched
// with launch() may have its CTAs made resident while its predecessor drains,
// so every such kernel first waits for the predecessor grid (and its memory)
// to complete; kernels whose CTAs all fit in one wave then let their own
// successor be launched at once (trigger), the rest at exit.
FS_DEVINL void pdl_entry(bool trigger) {
#if FS_WIDE_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

constexpr int kRadixBits = 8;
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;

// ---- k_scatter geometry
#ifndef FS_SCATTER_THREADS  // overridable for scripts/microbench/wide_variants.py
#define FS_SCATTER_THREADS 256
#define FS_SCATTER_ITEMS 16
#define FS_SCATTER_MINB 2
#endif
// Interleave groups (tickets run across G segments at a time): fewer concurrent
// write streams keep their partially written L2 lines resident (c5: level 2
// 4.04 -> 3.63 ms with 128 of its 256 segments, level 1 3.64 -> 3.58 ms with half
// of its chunks; 32 segments: 3.77 ms, the lookbacks start to wait).
#ifndef FS_L2_GROUP
#define FS_L2_GROUP 128
#endif
#ifndef FS_L1_HALVES
#define FS_L1_HALVES 1
#endif
// k_scatter reads its predecessor's status word early (1: when it publishes its
// own counts; 2: at tile start) and uses it at the lookback if it already held
// the inclusive prefix, saving the lookback's L2 round trip (0: off).
#ifndef FS_SCATTER_EARLY_LOOK
#define FS_SCATTER_EARLY_LOOK 1
#endif
#ifndef FS_SCATTER_L2PF  // k_scatter: bulk-prefetch the tile after next into L2 in these modes (bit mask)
#define FS_SCATTER_L2PF 4   // mode 2 (MSD level 2) only
#endif
#ifndef FS_SCATTER_STORE_UNROLL
#define FS_SCATTER_STORE_UNROLL 1
#endif
constexpr int kStoreUnroll = FS_SCATTER_STORE_UNROLL;
constexpr int kSThreads = FS_SCATTER_THREADS;
constexpr int kSWarps = kSThreads / 32;
constexpr int kSItems = FS_SCATTER_ITEMS;
constexpr int kSTile = kSThreads * kSItems;  // 4,096 keys per tile
constexpr int kSlack = 8;                    // 16-byte alignment slack of a tile buffer (elements)
static_assert(kSThreads >= kRadix, "one thread per digit in the lookback");

constexpr unsigned long long kStFlagAgg = 1ull << 62;
constexpr unsigned long long kStFlagInc = 2ull << 62;
constexpr int kTagShift = 56;
constexpr unsigned long long kStValue = (1ull << kTagShift) - 1;
constexpr uint32_t kNoTile = 0xFFFFFFFFu;

// ---- MSD geometry
constexpr int kTopBits = 16;            // bits binned by the trie (two 8-bit MSD levels)
constexpr int kSegs = 256;              // first-level segments
#ifndef FS_LOCAL_REHIST_INLINE
#define FS_LOCAL_REHIST_INLINE 0
#endif
#ifndef FS_LOCAL_THREADS
#define FS_LOCAL_THREADS 512
#endif
#ifndef FS_LOCAL_CB
#define FS_LOCAL_CB 12
#endif
// FS_RANK_PRED: the rank loop's conditional increment as one predicated add (4
// instructions per comparison instead of 5: the compiler's add + select): local
// sort 4.008 -> 3.985 ms at c5 (profiles/r02h/wide_variants_rank_pred.txt).
#ifndef FS_RANK_PRED
#define FS_RANK_PRED 1
#endif
#ifndef FS_RANK_MASKED
#define FS_RANK_MASKED 1
#endif
constexpr int kLocalThreads = FS_LOCAL_THREADS;
constexpr int kLocalCap = 8704;         // max keys of a 16-bit bin sorted in shared memory
constexpr int kIdxBits = 14;            // local index bits of the composite key
static_assert(kLocalCap <= (1 << kIdxBits), "local index must fit");
constexpr int kCountBitsMax = FS_LOCAL_CB;  // local counting digit (<= 4,096 groups)
#ifndef FS_RANK_U
#define FS_RANK_U 4
#endif
constexpr int kRankU = FS_RANK_U;       // keys ranked at once per thread (ILP)
// Fast path or slow path, per bin, from the counting digit's group sizes L_g:
// the rank loop costs ~ L per key (sum L_g^2 over the bin), the slow path a fixed
// number of multisplit passes; a bin takes the slow path if some group exceeds
// kMaxGroup or the key-weighted mean group size sum(L_g^2) / m exceeds
// kMeanGroupMax (repeated keys, 2^29 pairs, 16 copies of each key: local sort
// 25.5 -> 7.3 ms; profiles/r02d/wide_skew_dup.txt).  The slow path sorts by the
// counting digit first (two stable passes) and finishes groups of <=
// kGroupValuesMax distinct keys by value sweeps, else runs the full LSD.
#ifndef FS_MAX_GROUP
#define FS_MAX_GROUP 128
#endif
#ifndef FS_MEAN_GROUP
#define FS_MEAN_GROUP 48
#endif
constexpr int kMaxGroup = FS_MAX_GROUP;  // rank-loop bound of the fast path
constexpr int kMeanGroupMax = FS_MEAN_GROUP;
#ifndef FS_GROUP_VALUES_MAX  // slow path: most distinct keys in one group sorted by value sweeps (else the full LSD)
#define FS_GROUP_VALUES_MAX 16
#endif
constexpr int kGroupValuesMax = FS_GROUP_VALUES_MAX;
#ifndef FS_TINY_MAX  // bins of <= this many keys: one warp each (multiple of 32)
#define FS_TINY_MAX 128
#endif
#ifndef FS_SMALL_SORT_MSD_MAX  // one CTA (k_small_sort) up to this many keys when MSD could run
#define FS_SMALL_SORT_MSD_MAX 8960  // (pairs: 8,192 74 us vs 84 for MSD; 10,240: 91 vs 83)
#endif
#ifndef FS_MSD_MIN_N
#define FS_MSD_MIN_N (FS_SMALL_SORT_MSD_MAX + 1ull)
#endif
constexpr uint64_t kMsdMinN = FS_MSD_MIN_N;
constexpr uint32_t kTinyMax = FS_TINY_MAX;
constexpr int kMidCap = 2048;  // bins of kTinyMax+1 .. 2,048 keys: k_local_mid (smaller CTAs, 4 per SM)
constexpr uint64_t kListBigMaxN = 1ull << 26;  // below: k_local_sort runs from the plan's list of bins

struct LsdPlan {
  uint64_t base[kMaxPasses][kRadix];  // exclusive digit offsets
  uint32_t skip[kMaxPasses];
  uint32_t exec_index[kMaxPasses];    // 1-based index among executed passes
  uint32_t executed;                  // E
};

struct MsdPlan {
  uint32_t use_msd;           // 1: MSD kernels run, LSD kernels return; 0: the reverse
  uint32_t l2_tiles;          // tiles of the level-2 pass
  uint32_t l2_interleave;     // 1 (level 2 always interleaves: t -> r = t / 256, s = t % 256; buckets too
                              //    large for the status rows have 0 tiles here and run in k_heavy, level -1)
  uint32_t l2_rmax;           // most tiles in one segment
  int32_t kb;                 // key bits the MSD path bins: key_bits, or fewer above a common prefix
  uint32_t rehist;            // 1: the top-16 histogram is rebuilt on the window below the prefix
  uint32_t need_keybits;      // the first histogram has one bin: k_keybits looks at the keys
  uint64_t prefix;            // the keys' common bits above kb (0 if kb = key_bits)
  uint32_t seg_tile0[kSegs + 1];
  uint64_t seg_begin[kSegs + 1];
};

// ---- recursion into oversize bins (wide_heavy.cuh)
constexpr uint32_t kHeavyChunkKeys = 65536;  // target keys per chunk
constexpr uint32_t kHeavyMaxChunks = 1184;   // chunks per segment (bounds phase C's serial loops)
constexpr int kHeavyThreads = 256;           // = kRadix: thread d owns digit d
constexpr int kHeavyItems = 16;
constexpr int kHeavyTile = kHeavyThreads * kHeavyItems;
constexpr int kHeavyWarps = kHeavyThreads / 32;
constexpr int kHeavyMaxLevels = 6;           // (64 - 16) / 8

struct HeavySeg {
  uint64_t begin, count;
  uint32_t c0, nc;  // chunks [c0, c0 + nc) of the current level
  uint32_t buf;     // 0: the keys lie in the output, 1: in the temporary buffer
  uint32_t skip;    // every key has the same digit: not moved at this level
};

struct HeavyItem {
  uint64_t begin, count;
  uint64_t top;  // every key lies in [top, top + 2^R); sorted by key - top
  uint32_t R;    // 0: already in order, copy only
  uint32_t buf;  // where the keys lie
};
constexpr uint64_t kHeavyCopyPiece = 1ull << 20;  // copy items are emitted in pieces of this many keys

struct HeavyCtl {
  uint32_t nseg[2];                         // segments of the level with this parity
  uint32_t nl2;                             // segments of the uneven level-2 pass (level -1)
  uint32_t nchunks[kHeavyMaxLevels + 1];    // per level + 1
  uint32_t ticket[kHeavyMaxLevels + 1];
  uint32_t nitems;
  uint32_t ntiny;                           // bins of 2..kTinyMax keys (k_tiny_bins)
  uint32_t nbig;                            // bins for k_local_sort when it runs from a list (small inputs)
  uint32_t nmid;                            // bins of kTinyMax+1 .. kMidCap keys (k_local_mid)
  uint32_t one_bin;                         // one 16-bit bin holds every key (k_bin_lists)
};

struct HeavyCaps {
  uint64_t segs, chunks, items;
};

HeavyCaps heavy_caps(uint64_t n) {
  HeavyCaps c;
  c.segs = n / (kLocalCap + 1) + 1;
  c.chunks = n / kHeavyChunkKeys + c.segs + kSegs + 1;
  c.items = (uint64_t)kHeavyMaxLevels * (2 * (n / kLocalCap) + 2 * c.segs + 2 + n / kHeavyCopyPiece + c.segs) +
            kHistBins;  // + the 16-bit bins when the window moved below a common prefix
  return c;
}

template <typename K>
struct HeavyArgs {
  K* kout;
  uint32_t* vout;
  K* kalt;
  uint32_t* valt;
  uint64_t n;
  int tma;     // every buffer 16-byte aligned: bulk-copy tiles
  HeavyCtl* ctl;
  HeavySeg* segl2;  // level -1: the first-level buckets
  HeavySeg* seg0;  // segments of even levels
  HeavySeg* seg1;  // of odd levels
  uint32_t* chunk_seg;
  uint32_t* chist;      // [chunk][256]
  uint64_t* cbase;      // [chunk][256]
  HeavyItem* items;
  const MsdPlan* msd;
};


// Stable warp multisplit on an 8-bit digit: the lanes of `valid` holding the
// same digit as this lane.  Written in PTX so each bit costs setp + vote + selp
// + lop3 (the compiler's form of the same loop costs 6 instructions per bit;
// scripts/microbench/rank_bench.cu: 14.4 vs 24 cycles per warp-op per SM).
FS_DEVINL uint32_t match_digit8(uint32_t d, uint32_t valid) {
  uint32_t peers = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 v, m;\n\t"
        "and.b32 m, %1, %2;\n\tsetp.ne.u32 p, m, 0;\n\t"
        "vote.sync.ballot.b32 v, p, 0xffffffff;\n\t"
        "selp.b32 m, 0, -1, p;\n\t"
        "lop3.b32 %0, %0, v, m, 0x60;\n\t}"  // peers & (v ^ m): m = ~0 when the bit is 0
        : "+r"(peers)
        : "r"(d), "r"(1u << b));
  }
  return peers;
}

template <typename K>
FS_DEVINL uint32_t digit_of(K key, int shift) {
  return (uint32_t)(key >> shift) & (kRadix - 1);
}

FS_DEVINL bool lsd_enabled(const MsdPlan* msd) { return msd == nullptr || msd->use_msd == 0; }

// ================================================================ histograms
// LSD: all digit histograms from one read of the keys.
template <typename K>
__global__ void __launch_bounds__(512)
    k_digit_hist(const K* __restrict__ keys, uint64_t n, int passes, unsigned long long* __restrict__ hist,
                 const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!lsd_enabled(msd)) return;
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
    k_digit_plan(const unsigned long long* __restrict__ hist, uint64_t n, int passes, LsdPlan* __restrict__ plan,
                 const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!lsd_enabled(msd)) return;
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

// MSD: leaf level of the 16-level compressed trie over the top 16 key bits.
// Same counter layout and overflow protocol as hist16.cu: u16 counters packed
// two per word; an add whose returned word has a half >= 2^15 exchanges the word
// with 0 into the u64 spill.  Every add is checked at once: after a counter
// crosses 2^15 each thread adds at most one more key to it before exchanging it,
// and a warp's run add (lane 0) is at most 32 * kPerVec keys (64 for u64, 128 for
// u32 keys), so a counter stays below 2^15 + 32 warps x 32 * kPerVec + 1024 <
// 65,536 (static_assert in k_top16_hist).
constexpr uint32_t kHotMask = 0x80008000u;

// bm (shared): OR / OR-of-complement of the bins that spilled (their counters
// may read 0 at the flush although the bins are not empty).
FS_DEVINL void mark_bin(uint32_t* bm, uint32_t bin) {
  atomicOr(&bm[0], bin);
  atomicOr(&bm[1], ~bin & 0xFFFFu);
}

FS_DEVINL void top_add(uint32_t* sh, uint32_t bin, uint32_t cnt, unsigned long long* spill, uint32_t* l1spill,
                       uint32_t* bm) {
  const uint32_t w = bin >> 1;
  const uint32_t old = atomicAdd(&sh[w], (bin & 1u) ? (cnt << 16) : cnt);
  if (old & kHotMask) {
    const uint32_t x = atomicExch(&sh[w], 0u);
    if (x & 0xFFFFu) {
      atomicAdd(&spill[2 * w], (unsigned long long)(x & 0xFFFFu));
      mark_bin(bm, 2 * w);
    }
    if (x >> 16) {
      atomicAdd(&spill[2 * w + 1], (unsigned long long)(x >> 16));
      mark_bin(bm, 2 * w + 1);
    }
    if (x) atomicAdd(&l1spill[w >> 7], (x & 0xFFFFu) + (x >> 16));  // this chunk's level-1 count
  }
}

// CTA b histograms the contiguous chunk [b * chunk, (b+1) * chunk) of the keys,
// so its flushed partial is the chunk's own 16-bit histogram: the level-1
// scatter uses the chunks as virtual segments (k_vseg_counts / k_vseg_scan).
//
// First pass (msd == nullptr): the host's window [kb-16, kb).  Second pass (msd
// != nullptr): returns at once unless k_binbits / k_keybits asked for it to be
// rebuilt on the window below a common prefix (msd->rehist).
template <typename K>
__global__ void __launch_bounds__(1024, 1)
    k_top16_hist(const K* __restrict__ keys, uint64_t n, int shift, uint64_t chunk, uint32_t* __restrict__ partials,
                 unsigned long long* __restrict__ spill, uint32_t* __restrict__ l1spill,
                 unsigned long long* __restrict__ binbits, const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  constexpr int kPerVec = 16 / sizeof(K);
  constexpr int kUnroll = 4;
  static_assert((1u << 15) + 32u * 32u * kPerVec + 1024u < 65536u, "top16 spill bound violated");
  if (msd != nullptr) {
    if (!msd->rehist) return;
    shift = msd->kb - kTopBits;
  }
  extern __shared__ uint4 sm4[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(sm4);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  uint32_t* my_l1spill = l1spill + (uint64_t)blockIdx.x * kRadix;
  __shared__ uint32_t bm[2];
  if (tid < 2) bm[tid] = 0;
  for (int i = tid; i < kHistWords / 4; i += 1024) sm4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  const uint64_t c0 = (uint64_t)blockIdx.x * chunk, c1 = min(c0 + chunk, n);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(keys + c0);
  uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(K);
  if (head > c1 - c0) head = c1 - c0;
  const uint64_t nvec = (c1 - c0 - head) / kPerVec;
  const uint64_t tail0 = c0 + head + nvec * kPerVec;
  for (uint64_t t = tid; t < head + (c1 - tail0); t += 1024) {  // unaligned head and ragged tail
    const uint64_t idx = t < head ? c0 + t : tail0 + (t - head);
    top_add(sh, (uint32_t)(keys[idx] >> shift) & 0xFFFFu, 1u, spill, my_l1spill, bm);
  }
  const uint4* __restrict__ vec = reinterpret_cast<const uint4*>(keys + c0 + head);
  for (uint64_t it0 = 0; it0 < nvec; it0 += (uint64_t)kUnroll * 1024) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = it0 + u * 1024 + tid;
      v[u] = i < nvec ? ld_stream_v4(vec + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (it0 + u * 1024 + warp * 32 >= nvec) break;  // warp-uniform (warp vote inside)
      const bool valid = it0 + u * 1024 + tid < nvec;
      K k[kPerVec];
      memcpy(k, &v[u], 16);
      uint32_t b[kPerVec];
      bool same = valid;
#pragma unroll
      for (int j = 0; j < kPerVec; ++j) b[j] = (uint32_t)(k[j] >> shift) & 0xFFFFu;
      const uint32_t b0 = __shfl_sync(kFull, b[0], 0);
#pragma unroll
      for (int j = 0; j < kPerVec; ++j) same &= b[j] == b0;
      if (__ballot_sync(kFull, same) == kFull) {  // runs (sorted / low-entropy keys): one add per warp
        if (lane == 0) top_add(sh, b0, 32u * kPerVec, spill, my_l1spill, bm);
      } else if (valid) {
#pragma unroll
        for (int j = 0; j < kPerVec; ++j) top_add(sh, b[j], 1u, spill, my_l1spill, bm);
      }
    }
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(partials + (uint64_t)blockIdx.x * kHistWords);
  for (int i = tid; i < kHistWords / 4; i += 1024) dst[i] = sm4[i];
  if (binbits != nullptr && tid < 2 && bm[tid]) atomicOr(&binbits[tid], (unsigned long long)bm[tid]);  // spilled bins
}

// ---- the window of the MSD path (a common prefix of the keys)
// Bits where some keys differ decide the window: if the highest such bit hb is
// below key_bits - 1 (the keys share a prefix) and hb + 1 >= 32, the trie bins
// [hb - 15, hb] instead of the top 16 bits (the trie's depth only
// spans the bits that vary) and its histogram is rebuilt there; the prefix is
// put back on every key by the per-bin sort (k_heavy_items then sorts the
// bins).  First the bin indices of the first histogram: OR / OR-of-complement
// over the non-empty bins (k_binbits, whose last CTA decides); if they vary, hb
// lies in the window; if one bin holds every key, a pass over the keys finds hb
// (k_keybits, whose last CTA decides).  With fewer than 32 varying bits the LSD
// path (which skips uniform digits) is taken instead.
// Shared decision: varying bits -> the plan's window; zeroes the spills for the rebuild.
FS_DEVINL void set_window(MsdPlan* msd, int key_bits, unsigned long long varying, unsigned long long common,
                          unsigned long long* spill, uint32_t* l1spill, uint32_t l1spill_words, int* kb_sh) {
  if (threadIdx.x == 0) {
    const int kbe = varying ? 64 - __clzll((long long)varying) : 0;
    int kb = key_bits;
    uint64_t prefix = 0;
    if (kbe < key_bits && kbe >= 32) {
      kb = kbe;
      prefix = common & ~((1ull << kbe) - 1);
    }
    msd->kb = kb;
    msd->prefix = prefix;
    msd->rehist = kb != key_bits ? 1u : 0u;
    *kb_sh = kb;
  }
  __syncthreads();
  if (*kb_sh != key_bits) {  // the second histogram pass starts from zeroed spills
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) spill[i] = 0;
    for (uint32_t i = threadIdx.x; i < l1spill_words; i += blockDim.x) l1spill[i] = 0;
  }
}

constexpr int kBinbitsThreads = 256;

// OR / OR-of-complement of the non-empty bins over the first histogram's
// partials (+ the bins that spilled, marked by k_top16_hist); the last CTA
// decides the window, or asks k_keybits to look at the keys (one bin).
__global__ void __launch_bounds__(kBinbitsThreads)
    k_binbits(const uint32_t* __restrict__ partials, int rows, unsigned long long* __restrict__ bits,
              uint32_t* __restrict__ done, int key_bits, MsdPlan* __restrict__ msd,
              unsigned long long* __restrict__ spill, uint32_t* __restrict__ l1spill, uint32_t l1spill_words) {
  pdl_entry(true);
  const uint32_t w = blockIdx.x * kBinbitsThreads + threadIdx.x;  // counter word = bins 2w, 2w + 1
  uint32_t x = 0;
#pragma unroll 8
  for (int r = 0; r < rows; ++r) x |= __ldcg(partials + (uint64_t)r * kHistWords + w);
  uint32_t o = 0, no = 0;
  if (x & 0xFFFFu) { o |= 2 * w; no |= ~(2 * w) & 0xFFFFu; }
  if (x >> 16) { o |= 2 * w + 1; no |= ~(2 * w + 1) & 0xFFFFu; }
  o = __reduce_or_sync(kFull, o);
  no = __reduce_or_sync(kFull, no);
  if ((threadIdx.x & 31u) == 0 && (o | no)) {
    atomicOr(&bits[0], (unsigned long long)o);
    atomicOr(&bits[1], (unsigned long long)no);
  }
  __shared__ uint32_t last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ int kb_sh;
  const unsigned long long bo = __ldcg(&bits[0]), bn = __ldcg(&bits[1]);
  const int top = key_bits - kTopBits;
  if (threadIdx.x == 0) msd->need_keybits = (bo & bn) ? 0u : 1u;  // one bin: look at the keys
  set_window(msd, key_bits, (bo & bn) << top, bo << top, spill, l1spill, l1spill_words, &kb_sh);
}

template <typename K>
__global__ void __launch_bounds__(1024)
    k_keybits(const K* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ bits, uint32_t* __restrict__ done,
              int key_bits, MsdPlan* __restrict__ msd, unsigned long long* __restrict__ spill,
              uint32_t* __restrict__ l1spill, uint32_t l1spill_words) {
  pdl_entry(true);
  if (!msd->need_keybits) return;
  unsigned long long o = 0, no = 0;
  constexpr int kPerVec = 16 / sizeof(K);
  const uint64_t head0 = ((16 - ((uintptr_t)keys & 15)) & 15) / sizeof(K), head = head0 < n ? head0 : n;
  const uint64_t nvec = (n - head) / kPerVec, tail0 = head + nvec * kPerVec;
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = gt; i < head + (n - tail0); i += gs) {  // unaligned head and ragged tail
    const K k = keys[i < head ? i : tail0 + (i - head)];
    o |= k;
    no |= (K)~k;
  }
  const uint4* vec = reinterpret_cast<const uint4*>(keys + head);
  uint32_t oA = 0, oB = 0, nA = 0, nB = 0;  // word-wise: x, z = u64 low halves (u32: keys), y, w = high halves
#pragma unroll 4
  for (uint64_t i = gt; i < nvec; i += gs) {
    const uint4 q = ld_stream_v4(vec + i);
    oA |= q.x | q.z;
    oB |= q.y | q.w;
    nA |= ~q.x | ~q.z;
    nB |= ~q.y | ~q.w;
  }
  if (sizeof(K) == 8) {
    o |= ((unsigned long long)oB << 32) | oA;
    no |= ((unsigned long long)nB << 32) | nA;
  } else {
    o |= oA | oB;
    no |= nA | nB;
  }
  const uint32_t olo = __reduce_or_sync(kFull, (uint32_t)o), ohi = __reduce_or_sync(kFull, (uint32_t)(o >> 32));
  const uint32_t nlo = __reduce_or_sync(kFull, (uint32_t)no), nhi = __reduce_or_sync(kFull, (uint32_t)(no >> 32));
  if ((threadIdx.x & 31u) == 0) {
    atomicOr(&bits[0], ((unsigned long long)ohi << 32) | olo);
    atomicOr(&bits[1], ((unsigned long long)nhi << 32) | nlo);
  }
  // the last CTA to finish decides the window
  __shared__ uint32_t last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ int kb_sh;
  const unsigned long long mask = key_bits >= 64 ? ~0ull : ((1ull << key_bits) - 1);
  const unsigned long long ko = __ldcg(&bits[0]) & mask, kn = __ldcg(&bits[1]) & mask;
  set_window(msd, key_bits, ko & kn, ko, spill, l1spill, l1spill_words, &kb_sh);
}

constexpr uint32_t kVsegSplit = 8;
// Level-1 digit counts of every chunk: cnt[v][d] = sum of the chunk's 256 leaves
// under level-8 node d (its partial) + what the chunk spilled there.
__global__ void __launch_bounds__(256)
    k_vseg_counts(const uint32_t* __restrict__ partials, const uint32_t* __restrict__ l1spill,
                  uint32_t* __restrict__ cnt, const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!msd->use_msd) return;
  // kVsegSplit CTAs per chunk row, 256 / kVsegSplit digits each (one CTA per
  // row: 24 us of dependent L2 round trips even at small n)
  const uint32_t v = blockIdx.x / kVsegSplit, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t d0 = (blockIdx.x % kVsegSplit) * (kRadix / kVsegSplit);
  const uint4* row = reinterpret_cast<const uint4*>(partials + (uint64_t)v * kHistWords);
#pragma unroll
  for (uint32_t d = d0 + warp; d < d0 + kRadix / kVsegSplit; d += 8) {
    const uint4 q = __ldcg(row + d * 32 + lane);  // 128 words = 256 leaves
    uint32_t x = (q.x & 0xFFFFu) + (q.x >> 16) + (q.y & 0xFFFFu) + (q.y >> 16) + (q.z & 0xFFFFu) + (q.z >> 16) +
                 (q.w & 0xFFFFu) + (q.w >> 16);
    x = warp_sum(x);
    if (lane == 0) cnt[v * kRadix + d] = x + l1spill[v * kRadix + d];
  }
}

// vbase[v][d] = P16[d << 8] + sum_{v' < v} cnt[v'][d]: where chunk v's keys of
// level-1 digit d start in the level-1 output.  One warp per digit.
__global__ void __launch_bounds__(256)
    k_vseg_scan(const uint32_t* __restrict__ cnt, int nseg, const uint64_t* __restrict__ P16,
                uint64_t* __restrict__ vbase, const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!msd->use_msd) return;
  const uint32_t d = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
  uint64_t run = P16[d << 8];
  for (int v0 = 0; v0 < nseg; v0 += 32) {
    const int v = v0 + lane;
    const uint64_t c = v < nseg ? cnt[v * kRadix + d] : 0ull;
    const uint64_t inc = warp_inclusive_scan<uint64_t>(c);
    if (v < nseg) vbase[(uint64_t)v * kRadix + d] = run + inc - c;
    run += __shfl_sync(kFull, inc, 31);
  }
}

// The 16-bit bins, classified (many CTAs; every append is one atomic per CTA):
// above the local-sort capacity -> the recursion's first segments; 2..kTinyMax
// keys -> k_tiny_bins; ..kMidCap -> k_local_mid; the rest -> k_local_sort's list
// (small inputs only; large ones run one CTA per bin).  With a moved window
// (rehist) every bin of 2..cap keys becomes a k_heavy_items item instead.
constexpr int kListThreads = 256;
constexpr int kListBinsPerThread = 4;
constexpr int kListGrid = kHistBins / (kListThreads * kListBinsPerThread);  // 64

__global__ void __launch_bounds__(kListThreads)
    k_bin_lists(const uint64_t* __restrict__ H16, const uint64_t* __restrict__ P16, uint64_t n,
                const MsdPlan* __restrict__ plan, HeavyCtl* __restrict__ hctl, HeavySeg* __restrict__ hseg,
                HeavyItem* __restrict__ hitems, uint32_t* __restrict__ tiny, uint32_t* __restrict__ mid,
                uint32_t* __restrict__ big, int list_big) {
  pdl_entry(true);
  __shared__ uint32_t lsum[4][kListThreads / 32];
  __shared__ uint32_t lbase[4];
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t rehist = plan->rehist;
  const uint32_t R = (uint32_t)(plan->kb - kTopBits);
  uint64_t c[kListBinsPerThread];
  uint32_t v[kListBinsPerThread];
#pragma unroll
  for (int i = 0; i < kListBinsPerThread; ++i) {
    v[i] = blockIdx.x * (kListThreads * kListBinsPerThread) + i * kListThreads + t;
    c[i] = __ldg(H16 + v[i]);
  }
  uint32_t cls[kListBinsPerThread];  // 0 tiny, 1 mid, 2 big (listed), 3 item (rehist), 4 none
  uint32_t cnt[4] = {0, 0, 0, 0};
  bool one = false;
#pragma unroll
  for (int i = 0; i < kListBinsPerThread; ++i) {
    one |= c[i] == n;
    if (c[i] > (uint64_t)kLocalCap) hseg[atomicAdd(&hctl->nseg[0], 1u)] = HeavySeg{__ldg(P16 + v[i]), c[i], 0, 0, 0, 0};
    uint32_t k = 4;
    if (c[i] >= 2 && c[i] <= (uint64_t)kLocalCap) {
      if (rehist) k = 3;
      else if (c[i] <= kTinyMax) k = 0;
      else if (c[i] <= (uint64_t)kMidCap) k = 1;
      else if (list_big) k = 2;
    }
    cls[i] = k;
    if (k < 4) ++cnt[k];
  }
  if (one) hctl->one_bin = 1u;
  uint32_t off[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const uint32_t inc = warp_inclusive_scan<uint32_t>(cnt[l]);
    if (lane == 31) lsum[l][warp] = inc;
    off[l] = inc - cnt[l];
  }
  __syncthreads();
  if (t < 4) {  // one atomic per list and CTA
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kListThreads / 32; ++w) tot += lsum[t][w];
    uint32_t* ctr = t == 0 ? &hctl->ntiny : t == 1 ? &hctl->nmid : t == 2 ? &hctl->nbig : &hctl->nitems;
    lbase[t] = tot ? atomicAdd(ctr, tot) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int l = 0; l < 4; ++l) {
#pragma unroll
    for (int w = 0; w < kListThreads / 32; ++w)
      if (w < (int)warp) off[l] += lsum[l][w];
    off[l] += lbase[l];
  }
#pragma unroll
  for (int i = 0; i < kListBinsPerThread; ++i) {
    const uint32_t k = cls[i];
    if (k == 0) tiny[off[0]++] = v[i];
    else if (k == 1) mid[off[1]++] = v[i];
    else if (k == 2) big[off[2]++] = v[i];
    else if (k == 3 && !FS_LOCAL_REHIST_INLINE)
      hitems[off[3]++] = HeavyItem{__ldg(P16 + v[i]), c[i], plan->prefix | ((uint64_t)v[i] << R), R, 0};
  }
}

// MSD plan: the tiles of the level-2 pass (segments = first-level buckets,
// bounds from P16).  If one 16-bit bin holds all the keys (k_bin_lists: a common
// prefix the window could not move below) the LSD path runs instead, skipping
// its uniform digits.
__global__ void __launch_bounds__(kSegs)
    k_msd_plan(const uint64_t* __restrict__ P16, uint32_t status_cap, MsdPlan* __restrict__ plan,
               HeavyCtl* __restrict__ hctl, HeavySeg* __restrict__ hl2) {
  pdl_entry(true);
  __shared__ uint32_t wsum[kSegs / 32];
  __shared__ uint32_t rmax;
  const uint32_t s = threadIdx.x, lane = s & 31u, warp = s >> 5;
  if (s == 0) rmax = 0;
  __syncthreads();
  // Level 2: interleaved tickets (k_scatter mode 2) keep every bucket's lookback
  // one tile deep, but cost 256 x (most tiles in one bucket) status rows.  A
  // bucket above status_cap / 256 tiles (about 1.25x the mean) is left out of
  // the interleave (its tickets are holes) and run by k_heavy instead (chunk
  // histograms, CTA-owned chunks, no lookback).
  const uint64_t b = P16[s * 256], e = P16[(s + 1) * 256];
  const uint32_t all_tiles = (uint32_t)((e - b + kSTile - 1) / kSTile);
#ifdef FS_FORCE_L2_HEAVY  // timing experiment: level 2 always in k_heavy
  const bool to_heavy = e > b && status_cap;
#else
  const bool to_heavy = (uint64_t)all_tiles * kSegs > (uint64_t)status_cap;
#endif
  const uint32_t tiles = to_heavy ? 0u : all_tiles;
  if (to_heavy) hl2[atomicAdd(&hctl->nl2, 1u)] = HeavySeg{b, e - b, 0, 0, 1, 0};
  atomicMax(&rmax, tiles);
  const uint32_t inc = warp_inclusive_scan<uint32_t>(tiles);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSegs / 32; ++w) {
    if (w < (int)warp) off += wsum[w];
    tot += wsum[w];
  }
  plan->seg_tile0[s] = off + inc - tiles;
  plan->seg_begin[s] = b;
  if (s == kSegs - 1) {
    plan->seg_tile0[kSegs] = tot;
    plan->seg_begin[kSegs] = e;
    plan->l2_tiles = tot;
  }
  __syncthreads();
  if (s == 0) {
    plan->use_msd = __ldcg(&hctl->one_bin) ? 0u : 1u;
    plan->l2_rmax = rmax;
    plan->l2_interleave = 1u;
  }
}

// ================================================================ scatter pass
template <typename K>
struct ScatterArgs {
  const K* kin;             // the caller's input
  const uint32_t* vin;
  K* kA;                    // the caller's output
  uint32_t* vA;
  K* kB;                    // the temporary buffer
  uint32_t* vB;
  uint64_t n;
  int mode;                 // 0: LSD pass `pass`; 1: MSD level 1; 2: MSD level 2
  int pass;
  int shift;                // digit = (key >> shift) & 255
  const LsdPlan* lsd;
  const MsdPlan* msd;
  const uint64_t* P16;
  unsigned long long* status;
  uint32_t* ticket;
  unsigned long long tag;   // pass tag << kTagShift
  uint32_t tiles;           // ceil(n / kSTile)
  const uint64_t* vbase;    // mode 1: [chunk][digit] level-1 bases (k_vseg_scan)
  uint32_t l1_nseg;         // mode 1: chunks (virtual segments)
  uint32_t l1_chunk_tiles;  // mode 1: tiles per chunk
  int tma;                  // every buffer 16-byte aligned: bulk-copy prefetch
};

// Tile schedule.  Linear: ticket = tile index, the predecessor of a tile is the
// previous tile (mode 0).  Interleaved
// (modes 1, 2): ticket t is tile r = t / nseg of segment s = t % nseg, so the
// predecessor in the same segment was issued nseg tickets earlier and has
// normally published its inclusive prefix: lookbacks stay one round deep
// instead of trailing a single chain of ~10^5 tiles.  Status word index = ticket.
struct TileInfo {
  uint64_t begin, end, abeg;  // [begin, end) of the source; abeg = bulk-copy start (<= begin)
  uint32_t tile, seg;         // tile = ticket (kNoTile: no more work)
  uint32_t first;             // first tile of its segment
  uint32_t stride;            // ticket distance to the predecessor in the segment
};

template <typename K, bool kHasValues>
struct ScatterSmem {
  K keys[2][kSTile + kSlack];
  uint32_t vals[2][kHasValues ? kSTile + kSlack : 1];
  uint16_t whist[kSWarps][kRadix];   // per-warp counts, then per-warp offsets in the tile (<= 4096)
  uint32_t digit_start[kRadix];      // tile-local exclusive scan over digits
  unsigned long long gofs[kRadix];   // global offset - digit_start
  uint32_t seg_tile0[kSegs + 1];
  uint64_t seg_begin[kSegs + 1];
  uint32_t wsum[kRadix / 32];
  uint64_t mbar[2];
  TileInfo info[2];
};

template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kSThreads, FS_SCATTER_MINB) k_scatter(ScatterArgs<K> a) {
  pdl_entry(true);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<ScatterSmem<K, kHasValues>*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

  // ---- resolve this pass (uniform across the grid)
  const K* src_k;
  const uint32_t* src_v;
  K* dst_k;
  uint32_t* dst_v;
  const uint64_t* base_tab;
  uint32_t base_ss = 0, base_ds = 1, ntiles, nseg = 1;
  bool inter = false;
  if (a.mode == 0) {
    if (!lsd_enabled(a.msd) || a.lsd->skip[a.pass]) return;
    const uint32_t E = a.lsd->executed, e = a.lsd->exec_index[a.pass];
    const bool dst_is_a = ((E - e) & 1u) == 0;  // the last executed pass lands in the caller's output
    src_k = e == 1 ? a.kin : (dst_is_a ? a.kB : a.kA);
    src_v = e == 1 ? a.vin : (dst_is_a ? a.vB : a.vA);
    dst_k = dst_is_a ? a.kA : a.kB;
    dst_v = dst_is_a ? a.vA : a.vB;
    base_tab = a.lsd->base[a.pass];
    ntiles = a.tiles;
  } else {
    if (!a.msd->use_msd) return;
    if (a.mode == 1) {
      src_k = a.kin; src_v = a.vin; dst_k = a.kB; dst_v = a.vB;
      base_tab = a.vbase;
      base_ss = 256;  // level 1: base[v][d] = vbase[v * 256 + d]
      nseg = a.l1_nseg;
      inter = true;
      ntiles = a.l1_nseg * a.l1_chunk_tiles;
    } else {
      src_k = a.kB; src_v = a.vB; dst_k = a.kA; dst_v = a.vA;
      base_tab = a.P16;
      base_ss = 256;  // level 2: base[s][d] = P16[(s << 8) | d]
      inter = true;
      nseg = kSegs;
      ntiles = kSegs * a.msd->l2_rmax;
    }
  }
  const uint64_t n = a.n;
  const uint64_t n_al = n & ~(uint64_t)3;  // bulk copies never read past this

  // Tile of a ticket (shared-memory reads only): false for a hole.
  auto decode = [&](uint32_t tk, TileInfo& t) -> bool {
    t.tile = tk;
    t.stride = inter ? nseg : 1u;
    uint32_t r;
    uint64_t sb, se;
    if (inter) {
      t.seg = tk % nseg;
      r = tk / nseg;
#if FS_L2_GROUP < 256  // level 2 interleaves FS_L2_GROUP segments at a time (FS_L2_GROUP divides 256)
      if (a.mode == 2) {
        const uint32_t per = FS_L2_GROUP * a.msd->l2_rmax;
        t.seg = (tk % per) % FS_L2_GROUP + (tk / per) * FS_L2_GROUP;
        r = (tk % per) / FS_L2_GROUP;
        t.stride = FS_L2_GROUP;
      }
#endif
#if FS_L1_HALVES  // level 1 interleaves half of its chunks at a time (an even number of at least 64)
      if (a.mode == 1 && nseg % 2 == 0 && nseg >= 64) {
        const uint32_t g = nseg / 2, per = g * a.l1_chunk_tiles;
        t.seg = (tk % per) % g + (tk / per) * g;
        r = (tk % per) / g;
        t.stride = g;
      }
#endif
      if (a.mode == 1) {
        sb = (uint64_t)t.seg * a.l1_chunk_tiles * kSTile;
        se = min(sb + (uint64_t)a.l1_chunk_tiles * kSTile, n);
      } else {
        if (r >= sm.seg_tile0[t.seg + 1] - sm.seg_tile0[t.seg]) return false;  // segment has fewer tiles
        sb = sm.seg_begin[t.seg];
        se = sm.seg_begin[t.seg + 1];
      }
      if (sb + (uint64_t)r * kSTile >= se) return false;
    } else {
      t.seg = 0;
      r = tk;
      sb = 0;
      se = n;
    }
    t.first = r == 0;
    t.begin = sb + (uint64_t)r * kSTile;
    t.end = min(t.begin + (uint64_t)kSTile, se);
    t.abeg = a.tma ? (t.begin & ~(uint64_t)3) : t.begin;
    return true;
  };
  // Thread 0: take the next tile, describe it, and (with TMA) start its copy.
  // Tickets are requested one tile ahead (`spare`): the atomic's round trip
  // overlaps a whole tile instead of stalling thread 0 at every iteration.
  uint32_t spare = 0;
  auto fetch = [&](int buf) {
    TileInfo t;
    for (;;) {
      const uint32_t tk = spare;
      spare = atomicAdd(a.ticket, 1u);
      if (tk >= ntiles) {
        t.tile = kNoTile;
        t.begin = t.end = t.abeg = 0;
        t.seg = 0;
        t.first = 0;
        t.stride = 1;
        sm.info[buf] = t;
        return;
      }
      if (decode(tk, t)) break;
    }
    sm.info[buf] = t;
    if (a.tma) {
      const uint64_t aend = min((t.end + 3) & ~(uint64_t)3, n_al);
      const uint32_t cnt = aend > t.abeg ? (uint32_t)(aend - t.abeg) : 0u;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&sm.mbar[buf], cnt * (uint32_t)(sizeof(K) + (kHasValues ? 4 : 0)));
      if (cnt) {
        bulk_g2s(sm.keys[buf], src_k + t.abeg, cnt * (uint32_t)sizeof(K), &sm.mbar[buf]);
        if (kHasValues) bulk_g2s(sm.vals[buf], src_v + t.abeg, cnt * 4u, &sm.mbar[buf]);
      }
    }
  };
  // Thread 0: warm L2 with the tile after next (the spare ticket) so the bulk
  // copy issued for it one tile later finds its bytes on chip.
  auto prefetch_spare = [&]() {
    TileInfo t;
    if (!a.tma || spare >= ntiles || !decode(spare, t)) return;
    const uint64_t aend = min((t.end + 3) & ~(uint64_t)3, n_al);
    if (aend <= t.abeg) return;
    const uint32_t cnt = (uint32_t)(aend - t.abeg);
    bulk_prefetch_l2(src_k + t.abeg, cnt * (uint32_t)sizeof(K));
    if (kHasValues) bulk_prefetch_l2(src_v + t.abeg, cnt * 4u);
  };

  if (tid == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    mbar_fence_init();
  }
  if (a.mode == 2)
    for (int i = tid; i <= kSegs; i += kSThreads) {
      sm.seg_tile0[i] = __ldcg(&a.msd->seg_tile0[i]);
      sm.seg_begin[i] = __ldcg(&a.msd->seg_begin[i]);
    }
  for (int i = tid; i < kSWarps * kRadix / 2; i += kSThreads) reinterpret_cast<uint32_t*>(&sm.whist[0][0])[i] = 0;
  __syncthreads();
  if (tid == 0) {
    spare = atomicAdd(a.ticket, 1u);
    fetch(0);
  }
  __syncthreads();

  const int shift = a.mode == 0 ? a.shift : a.msd->kb - kRadixBits * a.mode;  // MSD: the plan's window
#ifdef FS_SCATTER_STATS
  long long ph_t0 = clock64();
#endif
  for (uint32_t it = 0;; ++it) {
    const int cur = it & 1;
    const TileInfo ti = sm.info[cur];
    if (ti.tile == kNoTile) break;
#ifndef FS_SCATTER_LATE_FETCH
    if (tid == 0) fetch(cur ^ 1);  // prefetch the next tile while this one is processed
#endif
    K* kbuf = sm.keys[cur];
    uint32_t* vbuf = kHasValues ? sm.vals[cur] : nullptr;
    const uint32_t len = (uint32_t)(ti.end - ti.begin);
    const uint32_t off = (uint32_t)(ti.begin - ti.abeg);
    if (a.tma) {
      mbar_wait(&sm.mbar[cur], (it >> 1) & 1u);
      // keys past the last 16-byte boundary of the array (< 4): plain loads
      const uint64_t covered = max(min((ti.end + 3) & ~(uint64_t)3, n_al), ti.begin);
      if (covered < ti.end) {
        const uint32_t e0 = (uint32_t)(covered - ti.begin);
        if (tid < len - e0) {
          kbuf[off + e0 + tid] = src_k[covered + tid];
          if (kHasValues) vbuf[off + e0 + tid] = src_v[covered + tid];
        }
        __syncthreads();
      }
    } else {
      for (uint32_t e = tid; e < len; e += kSThreads) {
        kbuf[e] = src_k[ti.begin + e];
        if (kHasValues) vbuf[e] = src_v[ti.begin + e];
      }
      __syncthreads();
    }

    // Digit threads fetch their global digit base now; it is needed only after the lookback.
    const uint32_t d = tid;
    const uint64_t dbase = d < kRadix ? __ldg(base_tab + (uint64_t)ti.seg * base_ss + (uint64_t)d * base_ds) : 0ull;
    unsigned long long pre = 0;  // the predecessor's status word, read early (FS_SCATTER_EARLY_LOOK)
#if FS_SCATTER_EARLY_LOOK == 2
    if (d < kRadix && !ti.first)
      pre = ld_relaxed_u64(a.status + (uint64_t)((int64_t)ti.tile - (int64_t)ti.stride) * kRadix + d);
#endif

    FS_PH(0);  // 0: fetch + wait for the tile's bytes
    // ---- items: warp w holds tile elements [256 w, 256 w + 256), item i of lane l = 256 w + 32 i + l
    K key[kSItems];
    uint32_t val[kHasValues ? kSItems : 1];
    const uint32_t e0 = warp * 32 * kSItems + lane;
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      const uint32_t e = e0 + 32 * i;
      key[i] = e < len ? kbuf[off + e] : K(0);
      if (kHasValues) val[i] = e < len ? vbuf[off + e] : 0u;
    }

    // ---- warp-level stable ranking (8-ballot multisplit)
    uint32_t rank[kSItems];
    uint16_t* wh = sm.whist[warp];
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      const bool valid = e0 + 32 * i < len;
      const uint32_t dg = digit_of(key[i], shift);
      const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
      const uint32_t leader = 31 - __clz(peers);
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = wh[dg];
        wh[dg] = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(kFull, old, leader);
      rank[i] = old + __popc(peers & lanemask_lt());
      __syncwarp();
    }
    __syncthreads();

    // L2 bulk prefetch of the tile after next, level 2 only (FS_SCATTER_L2PF: bit m
    // = pass mode m).  Round 1 measured it neutral everywhere; with the round-2
    // loop it costs level 1 ~0.09 ms per c5 sort (3.54 vs 3.45 ms without) but
    // helps level 2 on uneven buckets (16 hot bins: 2.70 vs 2.97 ms);
    // profiles/r02f/wide_variants_l2pf.txt.
    if (((FS_SCATTER_L2PF >> a.mode) & 1) && tid == 0) prefetch_spare();
    FS_PH(1);  // 1: load items + rank + barrier
    // ---- tile digit counts (thread = digit); publish; per-warp offsets
    uint32_t cnt = 0;
    unsigned long long* st = a.status + (uint64_t)ti.tile * kRadix + d;
#if FS_SCATTER_EARLY_LOOK == 1
    if (d < kRadix && !ti.first)
      pre = ld_relaxed_u64(a.status + (uint64_t)((int64_t)ti.tile - (int64_t)ti.stride) * kRadix + d);
#endif
    if (d < kRadix) {
#pragma unroll
      for (int w = 0; w < kSWarps; ++w) {
        const uint32_t c = sm.whist[w][d];
        sm.whist[w][d] = (uint16_t)cnt;
        cnt += c;
      }
      if (ti.first) st_relaxed_u64(st, kStFlagInc | a.tag | cnt);
      else st_relaxed_u64(st, kStFlagAgg | a.tag | cnt);
      const uint32_t inc = warp_inclusive_scan<uint32_t>(cnt);
      if (lane == 31) sm.wsum[warp] = inc;
      sm.digit_start[d] = inc - cnt;  // warp-local for now
    }
#ifdef FS_SCATTER_LATE_FETCH
    // The next ticket is taken only once this tile's counts are published: a
    // ticket held unstarted behind a busy tile would stall its successors'
    // lookbacks.
    if (tid == 0) fetch(cur ^ 1);
#endif
    __syncthreads();
    uint32_t dstart = 0;
    if (d < kRadix) {
#pragma unroll
      for (int w = 0; w < kRadix / 32; ++w)
        if (w < (int)warp) dstart += sm.wsum[w];
      dstart += sm.digit_start[d];
      sm.digit_start[d] = dstart;
#pragma unroll
      for (int w = 0; w < kSWarps; ++w) sm.whist[w][d] = (uint16_t)(sm.whist[w][d] + dstart);
    }
    __syncthreads();

    FS_PH(2);  // 2: counts, publish, digit scan, offsets (2 barriers)
    // ---- reorder through shared memory (the tile's input buffer becomes the stage)
#pragma unroll
    for (int i = 0; i < kSItems; ++i) {
      if (e0 + 32 * i < len) {
        const uint32_t pos = wh[digit_of(key[i], shift)] + rank[i];
        kbuf[pos] = key[i];
        if (kHasValues) vbuf[pos] = val[i];
      }
    }

    FS_PH(3);  // 3: reorder stores (thread 0's share)
    // ---- decoupled lookback over earlier tiles of the segment (thread = digit)
    if (d < kRadix) {
      unsigned long long excl = 0;
#ifdef FS_SCATTER_NOLOOKBACK  // timing experiment only: wrong offsets, no inter-tile dependency
      if (false) {
#else
      if (!ti.first) {
#endif
        const int64_t step = ti.stride;
        int64_t t = (int64_t)ti.tile - step;  // the segment's first tile publishes inclusive: the walk stops there
        // The immediate predecessor almost always holds its inclusive prefix by
        // now (scripts/microbench/scatter_stats.cu: 85-98%), so read it alone
        // first; a window of 8 older words only when it does not.  (Always
        // reading 8 rows cost ~16 KB of status traffic per tile, mostly DRAM:
        // the older rows have left L2.)
        bool done = false;
        {
          // the word read at publish time (one L2 round trip earlier) if it already
          // held the inclusive prefix, else a fresh read
          unsigned long long s = pre;
          if (!FS_SCATTER_EARLY_LOOK || (s & (0x3Full << kTagShift)) != a.tag || (s >> 62) != 2)
            s = ld_relaxed_u64(a.status + (uint64_t)t * kRadix + d);
          while ((s & (0x3Full << kTagShift)) != a.tag || (s >> 62) == 0)  // not yet published
            s = ld_relaxed_u64(a.status + (uint64_t)t * kRadix + d);
          excl += s & kStValue;
          done = (s >> 62) == 2;
          t -= step;
        }
        constexpr int kLook = 8;
        while (!done) {
          unsigned long long sv[kLook];
#pragma unroll
          for (int j = 0; j < kLook; ++j)
            sv[j] = t - j * step >= 0 ? ld_relaxed_u64(a.status + (uint64_t)(t - j * step) * kRadix + d)
                                      : (kStFlagInc | a.tag);
#pragma unroll
          for (int j = 0; j < kLook; ++j) {
            if (done) break;
            unsigned long long s = sv[j];
            while ((s & (0x3Full << kTagShift)) != a.tag || (s >> 62) == 0)  // not yet published
              s = ld_relaxed_u64(a.status + (uint64_t)(t - j * step) * kRadix + d);
            excl += s & kStValue;
            done = (s >> 62) == 2;
          }
          t -= kLook * step;
        }
        st_relaxed_u64(st, kStFlagInc | a.tag | (excl + cnt));
      }
      sm.gofs[d] = dbase + excl - dstart;
    }
    __syncthreads();

    FS_PH(4);  // 4: lookback + barrier
    // ---- scatter: consecutive positions of one digit go to consecutive addresses
#pragma unroll kStoreUnroll
    for (uint32_t j = tid; j < len; j += kSThreads) {
      const K k = kbuf[j];
      const uint64_t dst = sm.gofs[digit_of(k, shift)] + j;
      dst_k[dst] = k;
      if (kHasValues) dst_v[dst] = vbuf[j];
    }
    for (int i = tid; i < kSWarps * kRadix / 2; i += kSThreads) reinterpret_cast<uint32_t*>(&sm.whist[0][0])[i] = 0;
    FS_PH(5);  // 5: scatter stores (thread 0's share)
    __syncthreads();  // the stage (this buffer) is free for the prefetch after next
    FS_PH(6);  // 6: end barrier
  }
}

// If every LSD pass was skipped (all keys share every digit), the output is the input.
template <typename K, bool kHasValues>
__global__ void k_copy_if_identity(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
                                   uint32_t* __restrict__ vout, uint64_t n, const LsdPlan* __restrict__ plan,
                                   const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  if (!lsd_enabled(msd) || plan->executed != 0) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    kout[i] = kin[i];
    if (kHasValues) vout[i] = vin[i];
  }
}

// ================================================================ local sort
// One CTA per 16-bit bin b = [P16[b], P16[b+1]) of the output (in place): the
// L2 bulk prefetch of the 16-byte-aligned part of [b, e) (never beyond it).
FS_DEVINL void prefetch_l2_range(const void* b, const void* e) {
  const uintptr_t lo = ((uintptr_t)b + 15) & ~(uintptr_t)15, hi = (uintptr_t)e & ~(uintptr_t)15;
  for (uintptr_t a = lo; a < hi; a += 65536) {
    const uintptr_t len = hi - a < 65536 ? hi - a : 65536;
    bulk_prefetch_l2((const void*)a, (uint32_t)len);
  }
}

// 1 or 0x10000 by the low bit of g: the increment of the packed u16 counter pair
// word g >> 1.  FS_HALF_INC_MAD: one IMAD (g & 1) * 0xFFFF + 1, kept opaque to the
// compiler's rewrite into compare + select (local sort 3.985 -> 3.973 ms at c5,
// profiles/r02i/wide_variants_half_inc.txt).
#ifndef FS_HALF_INC_MAD
#define FS_HALF_INC_MAD 1
#endif
FS_DEVINL uint32_t half_inc(uint32_t g) {
#if FS_HALF_INC_MAD
  uint32_t r;
  asm("mad.lo.u32 %0, %1, 65535, 1;" : "=r"(r) : "r"(g & 1u));
  return r;
#else
  return (g & 1u) ? 0x10000u : 1u;
#endif
}

// Geometry of one per-bin sort: kThreads (>= 256: the slow path's digit scan
// uses one thread per digit) and the largest bin kCap.
template <int kThreads_, int kCap_>
struct LocalCfg {
  static constexpr int kThreads = kThreads_, kWarps = kThreads_ / 32, kCap = kCap_;
  static constexpr int kPer = (kCap + kThreads - 1) / kThreads;  // composites per thread
  static_assert(kThreads >= kRadix, "one thread per digit in the slow path");
  static_assert(kCap <= (1 << kIdxBits), "local index must fit");
};
using BigCfg = LocalCfg<kLocalThreads, kLocalCap>;  // 16-bit bins up to 8,704 keys, 2 CTAs per SM
using MidCfg = LocalCfg<256, kMidCap>;             // bins of kTinyMax+1 .. kMidCap keys, 4 CTAs per SM

template <class Cfg>
struct LocalLayout {
  static constexpr int ck = 0;                                      // u64[kCap]
  static constexpr int perm = ck + Cfg::kCap * 8;                   // u16[kCap]
  static constexpr int scratch = perm + Cfg::kCap * 2;
  // fast path: counters u16[2^kCountBitsMax]; the final permutation lives in `perm`
  // slow path: perm_b u16[kCap], then per-warp digit offsets u16[warps][256]
  static constexpr int perm_b = scratch;
  static constexpr int whist = scratch + Cfg::kCap * 2;
  static constexpr int fast_end = scratch + (1 << kCountBitsMax) * 2;
  static constexpr int slow_end = whist + Cfg::kWarps * kRadix * 2;
  static constexpr int total = fast_end > slow_end ? fast_end : slow_end;
};
using LocalSmemLayout = LocalLayout<BigCfg>;
static_assert(LocalSmemLayout::total <= 113 * 1024, "two CTAs per SM");

// per-bin sort of Alg. 5 ("sort_bin"), stable: every key of
// the bin lies in [top, top + 2^R) (a 16-bit bin: top = bin << R, R = key_bits -
// 16; a recursion item: see wide_heavy.cuh) and is ordered by its offset
// key - top.  Keys become composites c = (key - top) << 14 | i
// (i = arrival index inside the bin), all distinct, so ordering composites is
// the stable order.
//  counting sort by the top `cb` of the R bits (cb = ceil(log2 m), <= 12;
//    groups of ~1-2 keys for distinct keys) with shared atomics; then, chosen
//    per bin from the group sizes (kMaxGroup, kMeanGroupMax):
//  fast path: every key's final position = group start + #composites of its
//    group below its own;
//  slow path (large groups: repeated keys, low-entropy bins): stable passes by
//    the counting digit on a permutation (warp multisplit ranks), after which a
//    group of one value is final and a group of <= kGroupValuesMax values is
//    finished by value sweeps; otherwise a stable LSD over the varying 8-bit
//    digits of the R bits.
// Output: kout[b0 + j] = top + (c_j >> 14), vout[b0 + j] = vin[b0 + i_j]; kin == kout
// (in place) is allowed: every key is in registers before the first store.
template <typename K, bool kHasValues, class Cfg = BigCfg>
__device__ __forceinline__ void sort_bin(const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, uint64_t b0,
                                         uint32_t m, int R, K top) {
  using Lay = LocalLayout<Cfg>;
  constexpr int kLocalThreads = Cfg::kThreads, kLocalWarps = Cfg::kWarps, kLocalCap = Cfg::kCap;
  (void)kLocalCap;
#ifdef FS_SCATTER_STATS
  long long lph_t0 = clock64();
#endif
  // The values are read only after the key phases: start pulling them into L2
  // now (4.38 vs 4.41 ms at c5; prefetching the bin one wave ahead did nothing).
  if (kHasValues && threadIdx.x == 0) prefetch_l2_range(vin + b0, vin + b0 + m);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* ck = reinterpret_cast<uint64_t*>(smem_raw + Lay::ck);
  uint16_t* perm = reinterpret_cast<uint16_t*>(smem_raw + Lay::perm);
  uint32_t* cntw = reinterpret_cast<uint32_t*>(smem_raw + Lay::scratch);
  uint16_t* cnt16 = reinterpret_cast<uint16_t*>(cntw);
  __shared__ uint32_t heavy, s_sq, s_maxl, s_fallback;
  __shared__ uint32_t wtot[kLocalWarps];
  __shared__ unsigned long long or_all, and_all;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

  // counting digit: top cb of the R bits, cb = ceil(log2 m) capped
  int cb = 32 - __clz(m - 1);
  cb = min(cb, min(kCountBitsMax, R));
  const uint32_t ngroups = 1u << cb;
  const uint32_t nwords = (ngroups + 1) >> 1;
  const int cshift = kIdxBits + R - cb;

  if (tid == 0) heavy = s_sq = s_maxl = 0;
  // Keys: all loads in flight at once, turned into composites that stay in
  // registers; the digit histogram is counted from them; after the scan each
  // composite is written straight to its group's slot (ck is filled in group
  // order, never in arrival order: the arrival index is in the composite).
  constexpr int kPer = Cfg::kPer;  // 17 (big), 8 (mid)
  uint64_t cr[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t i = tid + u * kLocalThreads;
    cr[u] = i < m ? (((uint64_t)(kin[b0 + i] - top)) << kIdxBits) | i : 0ull;
  }
  for (uint32_t w = tid; w < nwords; w += kLocalThreads) cntw[w] = 0;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t i = tid + u * kLocalThreads;
    if (i < m) {
      const uint32_t g = (uint32_t)(cr[u] >> cshift) & (ngroups - 1);
      atomicAdd(&cntw[g >> 1], half_inc(g));
    }
  }
  __syncthreads();

  FS_LPH(0);  // 0: key loads + composites + histogram atomics (+2 barriers)
  // ---- exclusive scan of the ngroups counters (thread t: words [t*wpt, (t+1)*wpt))
#ifndef FS_LOCAL_VSCAN
#define FS_LOCAL_VSCAN 1
#endif
  if (FS_LOCAL_VSCAN && nwords == 4u * kLocalThreads) {
    // the common full-size case (4,096 groups, 512 threads; 2,048 / 256 for the
    // mid bins): each thread's four words are one 16-byte shared load and store
    // (four scalar loads at a 4-word stride were 4-way bank conflicts each)
    uint4* cw4 = reinterpret_cast<uint4*>(cntw);
    const uint4 x = cw4[tid];
    const uint32_t a0 = (x.x & 0xFFFFu), a1 = (x.x >> 16), b0 = (x.y & 0xFFFFu), b1 = (x.y >> 16);
    const uint32_t c0 = (x.z & 0xFFFFu), c1 = (x.z >> 16), d0 = (x.w & 0xFFFFu), d1 = (x.w >> 16);
    const uint32_t local = a0 + a1 + b0 + b1 + c0 + c1 + d0 + d1;
    const uint32_t sq = a0 * a0 + a1 * a1 + b0 * b0 + b1 * b1 + c0 * c0 + c1 * c1 + d0 * d0 + d1 * d1;
    const uint32_t mx = max(max(max(a0, a1), max(b0, b1)), max(max(c0, c1), max(d0, d1)));
    const uint32_t wsq = __reduce_add_sync(kFull, sq), wmx = __reduce_max_sync(kFull, mx);
    if (lane == 0) {
      atomicAdd(&s_sq, wsq);
      atomicMax(&s_maxl, wmx);
    }
    const uint32_t inc = warp_inclusive_scan<uint32_t>(local);
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    uint32_t run = inc - local;
    for (int w = 0; w < (int)warp; ++w) run += wtot[w];
    uint4 y;
    y.x = run | ((run + a0) << 16);
    run += a0 + a1;
    y.y = run | ((run + b0) << 16);
    run += b0 + b1;
    y.z = run | ((run + c0) << 16);
    run += c0 + c1;
    y.w = run | ((run + d0) << 16);
    cw4[tid] = y;
  } else {
    const uint32_t wpt = (nwords + kLocalThreads - 1) / kLocalThreads;  // <= 8
    const uint32_t w0 = tid * wpt;
    uint32_t local = 0, sq = 0, mx = 0;
    for (uint32_t j = 0; j < wpt; ++j)
      if (w0 + j < nwords) {
        const uint32_t x = cntw[w0 + j], lo = x & 0xFFFFu, hi = x >> 16;
        local += lo + hi;
        sq += lo * lo + hi * hi;
        mx = max(mx, max(lo, hi));
      }
    const uint32_t wsq = __reduce_add_sync(kFull, sq), wmx = __reduce_max_sync(kFull, mx);
    if (lane == 0) {
      atomicAdd(&s_sq, wsq);
      atomicMax(&s_maxl, wmx);
    }
    const uint32_t inc = warp_inclusive_scan<uint32_t>(local);
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    uint32_t run = inc - local;
    for (int w = 0; w < (int)warp; ++w) run += wtot[w];
    for (uint32_t j = 0; j < wpt; ++j)
      if (w0 + j < nwords) {
        const uint32_t x = cntw[w0 + j];
        const uint32_t lo = run, hi = run + (x & 0xFFFFu);
        run = hi + (x >> 16);
        cntw[w0 + j] = lo | (hi << 16);
      }
  }
  __syncthreads();
  // (read by every thread after the counting scatter's barrier)
  if (tid == 0 && (s_maxl > (uint32_t)kMaxGroup || s_sq > (uint32_t)kMeanGroupMax * m)) heavy = 1;

  FS_LPH(1);  // 1: scan
  // ---- counting scatter of the composites (order inside a group is fixed below)
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t i = tid + u * kLocalThreads;
    if (i < m) {
      const uint32_t g = (uint32_t)(cr[u] >> cshift) & (ngroups - 1);
      const uint32_t old = atomicAdd(&cntw[g >> 1], half_inc(g));
      ck[(g & 1u) ? (old >> 16) : (old & 0xFFFFu)] = cr[u];
    }
  }
  __syncthreads();

  FS_LPH(2);  // 2: counting scatter
  // ---- final positions: group start + rank of the composite inside its group
  //      (cnt16[g] = end of group g); fin[position] = the composite's ck slot,
  //      so the keys are written out coalesced after the barrier.
  uint16_t* fin = perm;
  // kRankU keys per thread at once: their group scans are independent shared
  // loads, interleaved (the loop runs to the longest of the kRankU groups).
  // (Measured at c5: 4.41 ms vs 4.50 for one key at a time with the keys
  // stored from here, 4.74 for one at a time staged, 5.34 for kRankU = 8; an
  // insertion sort per group, one thread per group: 5.15.)
  for (uint32_t j0 = heavy ? m : tid; j0 < m; j0 += kRankU * kLocalThreads) {  // slow-path bins skip the ranks
    uint64_t c[kRankU];
    uint32_t s[kRankU], e[kRankU], r[kRankU];
    uint32_t len = 0;
#pragma unroll
    for (int u = 0; u < kRankU; ++u) {
      const uint32_t j = j0 + u * kLocalThreads;
      c[u] = j < m ? ck[j] : 0ull;
      const uint32_t g = (uint32_t)(c[u] >> cshift) & (ngroups - 1);
      s[u] = g ? cnt16[g - 1] : 0u;
      e[u] = j < m ? (uint32_t)cnt16[g] : s[u];
      r[u] = s[u];
      len = max(len, e[u] - s[u]);
    }
    if (len > (uint32_t)kMaxGroup) continue;  // never: such a bin was sent to the slow path above
#if FS_RANK_MASKED
    // branch-free: every key reads len entries from its group start and masks the
    // ones past its group.  The reads stay inside the shared layout (s + len <= m
    // + kMaxGroup, and perm, kCap u16, follows ck); an entry read past the group
    // may be a perm slot another thread is writing -- its value is masked out.
    static_assert(Cfg::kCap * 2 >= kMaxGroup * 8, "over-reads of ck stay inside perm");
    uint32_t nu[kRankU];
#pragma unroll
    for (int u = 0; u < kRankU; ++u) nu[u] = e[u] - s[u];
    for (uint32_t k = 0; k < len; ++k) {
#pragma unroll
      for (int u = 0; u < kRankU; ++u) {
#if FS_RANK_PRED  // one predicated add (setp.lt.u64, setp.and, @p add) instead of add + select
        const uint64_t e = ck[s[u] + k];
        asm("{\n\t.reg .pred p;\n\tsetp.lt.u64 p, %1, %2;\n\tsetp.lt.and.u32 p, %3, %4, p;\n\t@p add.u32 %0, %0, 1;\n\t}"
            : "+r"(r[u])
            : "l"(e), "l"(c[u]), "r"(k), "r"(nu[u]));
#else
        r[u] += (uint32_t)((ck[s[u] + k] < c[u]) & (k < nu[u]));
#endif
      }
    }
#else
    for (uint32_t k = 0; k < len; ++k) {
#pragma unroll
      for (int u = 0; u < kRankU; ++u)
        if (s[u] + k < e[u]) r[u] += ck[s[u] + k] < c[u];
    }
#endif
#pragma unroll
    for (int u = 0; u < kRankU; ++u)
      if (j0 + u * kLocalThreads < m) fin[r[u]] = (uint16_t)(j0 + u * kLocalThreads);
  }
  __syncthreads();

  FS_LPH(3);  // 3: ranks
  uint16_t* pfinal = fin;
  if (heavy) {
    // ---- slow path: stable LSD over the varying 8-bit digits of the R bits
    uint16_t* pa = perm;
    uint16_t* pb = reinterpret_cast<uint16_t*>(smem_raw + Lay::perm_b);
    uint16_t* wh16 = reinterpret_cast<uint16_t*>(smem_raw + Lay::whist);  // [warp][digit]
    if (tid == 0) {
      or_all = 0;
      and_all = ~0ull;
    }
    __syncthreads();
    unsigned long long o = 0, an = ~0ull;
    for (uint32_t j = tid; j < m; j += kLocalThreads) {  // ck is in group order: pa lists it in arrival order
      const uint64_t c = ck[j];
      const uint64_t v = c >> kIdxBits;
      o |= v;
      an &= v;
      pa[c & ((1u << kIdxBits) - 1)] = (uint16_t)j;
    }
    atomicOr(&or_all, o);
    atomicAnd(&and_all, an);
    __syncthreads();
    const uint64_t varying = or_all ^ and_all;
    const uint32_t chunk = ((m + kLocalWarps - 1) / kLocalWarps + 31) & ~31u;
    const uint32_t c0 = min(warp * chunk, m), c1 = min(c0 + chunk, m);
    // One stable pass pa -> pb by the digit (ck[p] >> shift) & dmask (dmask <= 255).
    auto lsd_pass = [&](int shift, uint32_t dmask) {
      for (int i = tid; i < kLocalWarps * kRadix; i += kLocalThreads) wh16[i] = 0;
      __syncthreads();
      uint16_t* whw = wh16 + warp * kRadix;
      // pass A: per-warp digit counts over the warp's chunk
      for (uint32_t j0 = c0; j0 < c1; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool valid = j < c1;
        const uint32_t dg = valid ? (uint32_t)(ck[pa[j]] >> shift) & dmask : 0u;
        const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
        if (valid && lane == 31 - __clz(peers)) whw[dg] = (uint16_t)(whw[dg] + __popc(peers));
        __syncwarp();
      }
      __syncthreads();
      // scan over (digit major, warp minor): thread d < 256 owns digit d
      if (tid < kRadix) {
        uint32_t tot = 0;
        for (int w = 0; w < kLocalWarps; ++w) tot += wh16[w * kRadix + tid];
        const uint32_t inc = warp_inclusive_scan<uint32_t>(tot);
        if (lane == 31) wtot[warp] = inc;
      }
      __syncthreads();
      if (tid < kRadix) {
        uint32_t tot = 0;
        for (int w = 0; w < kLocalWarps; ++w) tot += wh16[w * kRadix + tid];
        uint32_t run = warp_inclusive_scan<uint32_t>(tot) - tot;
        for (int w = 0; w < (int)warp; ++w) run += wtot[w];
        for (int w = 0; w < kLocalWarps; ++w) {
          const uint32_t c = wh16[w * kRadix + tid];
          wh16[w * kRadix + tid] = (uint16_t)run;
          run += c;
        }
      }
      __syncthreads();
      // pass B: stable ranks, scatter of the permutation
      for (uint32_t j0 = c0; j0 < c1; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool valid = j < c1;
        const uint16_t p = valid ? pa[j] : (uint16_t)0;
        const uint32_t dg = valid ? (uint32_t)(ck[p] >> shift) & dmask : 0u;
        const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
        const uint32_t leader = 31 - __clz(peers);
        uint32_t old = 0;
        if (valid && lane == leader) {
          old = whw[dg];
          whw[dg] = (uint16_t)(old + __popc(peers));
        }
        old = __shfl_sync(kFull, old, leader);
        if (valid) pb[old + __popc(peers & lanemask_lt())] = p;
        __syncwarp();
      }
      __syncthreads();
      uint16_t* t = pa;
      pa = pb;
      pb = t;
    };
    bool done = false;
#ifndef FS_GROUP_FIRST
#define FS_GROUP_FIRST 1
#endif
    if (FS_GROUP_FIRST && ngroups > 1) {
      // Group digit first: two stable passes by the counting digit put every group
      // in arrival order, so a group whose keys are all equal (repeated keys) is
      // already sorted; a group of a few values (<= kGroupValuesMax) is ordered by
      // one stable compaction sweep per value; more values send the bin to the
      // full LSD over the varying digits.
      const int gb = cb < 8 ? cb : 8;
      lsd_pass(cshift, (1u << gb) - 1u);
      if (cb > 8) lsd_pass(cshift + 8, (1u << (cb - 8)) - 1u);
#if FS_GROUP_FIRST == 2  // timing experiment only: assume every group holds one value
      pfinal = pa;
      done = true;
      if (false)
#endif
      {
      if (tid == 0) s_fallback = 0;
      __syncthreads();
      // Group boundaries (the counters under perm_b are gone): a group starts where
      // the digit changes along pa.  A warp handles the groups that start in its
      // chunk [c0, c1), scanning past c1 for the end of its last one.
      auto gof = [&](uint32_t q) -> uint32_t { return (uint32_t)(ck[pa[q]] >> cshift) & (ngroups - 1u); };
      auto handle = [&](uint32_t gs, uint32_t ge) {  // warp-wide
        uint64_t mn = ~0ull, mx = 0;
        for (uint32_t q = gs + lane; q < ge; q += 32) {
          const uint64_t kp = ck[pa[q]] >> kIdxBits;
          mn = kp < mn ? kp : mn;
          mx = kp > mx ? kp : mx;
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
          const uint64_t a = __shfl_xor_sync(kFull, mn, d), b = __shfl_xor_sync(kFull, mx, d);
          mn = a < mn ? a : mn;
          mx = b > mx ? b : mx;
        }
        if (mn == mx) {  // one value: arrival order is the order
          for (uint32_t q = gs + lane; q < ge; q += 32) pb[q] = pa[q];
          return;
        }
        // a few values: one stable compaction sweep per value, smallest first
        // (the group is in arrival order); more than kGroupValuesMax values: the
        // bin takes the full LSD
        uint64_t cur = mn;
        uint32_t base = gs;
        for (int it = 0;; ++it) {
          if (it == kGroupValuesMax) {
            if (lane == 0) s_fallback = 1;
            return;
          }
          uint64_t nxt = ~0ull;
          for (uint32_t q0 = gs; q0 < ge; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint64_t kp = q < ge ? ck[pa[q]] >> kIdxBits : ~0ull;
            const bool eq = q < ge && kp == cur;
            const uint32_t bal = __ballot_sync(kFull, eq);
            if (eq) pb[base + __popc(bal & lanemask_lt())] = pa[q];
            base += __popc(bal);
            nxt = (kp > cur && kp < nxt) ? kp : nxt;
          }
#pragma unroll
          for (int d = 16; d >= 1; d >>= 1) {
            const uint64_t a = __shfl_xor_sync(kFull, nxt, d);
            nxt = a < nxt ? a : nxt;
          }
          if (nxt == ~0ull) return;
          cur = nxt;
        }
      };
      if (c0 < c1) {
        constexpr uint32_t kNone = 0xFFFFFFFFu;
        uint32_t open = kNone;                               // start of the group being scanned
        uint32_t gprev = c0 > 0 ? gof(c0 - 1) : kNone;       // digit just before this block
        bool stop = false;
        for (uint32_t q0 = c0; q0 <= m && !stop; q0 += 32) {
          const uint32_t q = q0 + lane;
          const uint32_t gq = q < m ? gof(q) : 0xFFFFFFFEu;  // position m closes the last group
          uint32_t gl = __shfl_up_sync(kFull, gq, 1);
          if (lane == 0) gl = gprev;
          uint32_t starts = __ballot_sync(kFull, q <= m && gq != gl);
          gprev = __shfl_sync(kFull, gq, 31);
          while (starts) {
            const uint32_t t = q0 + (uint32_t)(__ffs(starts) - 1);
            starts &= starts - 1;
            if (open != kNone) handle(open, t);
            open = kNone;
            if (t < c1 && t < m) {
              open = t;
            } else {
              stop = true;
              break;
            }
          }
        }
      }
      __syncthreads();
      if (!s_fallback) {
        pfinal = pb;
        done = true;
      } else {  // back to arrival order for the full LSD
        for (uint32_t j = tid; j < m; j += kLocalThreads) pa[ck[j] & ((1u << kIdxBits) - 1)] = (uint16_t)j;
        __syncthreads();
      }
      }
    }
    if (!done) {
      for (int sh = 0; sh < R; sh += kRadixBits) {
        if (((varying >> sh) & 0xFFu) == 0) continue;  // uniform digit: the pass is the identity
        lsd_pass(kIdxBits + sh, 0xFFu);
      }
      pfinal = pa;
    }
  }

  FS_LPH(4);  // 4: slow path (heavy bins only)
  // ---- write the bin back in sorted order: pfinal lists ck slots; write the
  //      keys, then turn it into arrival indices for the values
  {
#pragma unroll 4
    for (uint32_t j = tid; j < m; j += kLocalThreads) {
      const uint64_t c = ck[pfinal[j]];
      kout[b0 + j] = top + (K)(c >> kIdxBits);
      pfinal[j] = (uint16_t)(c & ((1u << kIdxBits) - 1));
    }
  }
  if (kHasValues) {
    __syncthreads();  // ck is free: stage the values there (arrival order)
    uint32_t* sv = reinterpret_cast<uint32_t*>(ck);
    // (Loading these right after the counting scatter, in flight during the
    // ranks, measured 4.61 vs 4.38 ms.)
    uint32_t vr[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t i = tid + u * kLocalThreads;
      vr[u] = i < m ? vin[b0 + i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t i = tid + u * kLocalThreads;
      if (i < m) sv[i] = vr[u];
    }
    __syncthreads();
    for (uint32_t j = tid; j < m; j += kLocalThreads) vout[b0 + j] = sv[pfinal[j]];
  }
  FS_LPH(5);  // 5: values
}

// One CTA per 16-bit bin of the MSD path, in place in the output.  Bins above
// the capacity are left to the recursion (k_heavy).
template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kLocalThreads, 2)
    k_local_sort(K* __restrict__ keys, uint32_t* __restrict__ vals, const uint64_t* __restrict__ P16, int R,
                 const MsdPlan* __restrict__ msd, const uint32_t* __restrict__ big, const HeavyCtl* __restrict__ ctl) {
  pdl_entry(false);
  // (R is the host's key_bits - 16.  A window moved below a common prefix sends
  // every bin to k_heavy_items instead: a loaded R costs ~26 us here at c5 — it
  // takes a register where the kernel parameter is an operand.)
  const uint32_t use = __ldg(&msd->use_msd), rehist = __ldg(&msd->rehist);
  if (!use) return;
  uint32_t bkt = blockIdx.x;
  if (big != nullptr) {  // small inputs: one CTA per listed bin, not one per bin
    if (bkt >= __ldg(&ctl->nbig)) return;
    bkt = __ldg(big + bkt);
  }
  const uint64_t b0 = __ldg(P16 + bkt);
  const uint32_t m = (uint32_t)(__ldg(P16 + bkt + 1) - b0);
  if (m <= (uint32_t)kMidCap || m > (uint32_t)kLocalCap) return;  // tiny / mid bins: their own kernels
#if FS_LOCAL_REHIST_INLINE
  if (rehist) {  // the window moved below a common prefix: the plan's R and prefix
    const int Rw = __ldg(&msd->kb) - kTopBits;
    sort_bin<K, kHasValues>(keys, vals, keys, vals, b0, m, Rw, (K)(__ldg(&msd->prefix) | ((uint64_t)bkt << Rw)));
    return;
  }
#else
  if (rehist) return;
#endif
  sort_bin<K, kHasValues>(keys, vals, keys, vals, b0, m, R, (K)((uint64_t)bkt << R));
}


// Bins of kTinyMax+1 .. kMidCap keys: the same per-bin sort with 256 threads and
// a 2,048-key shared layout, so four bins are in flight per SM instead of two.
// One CTA per listed bin (small inputs) or a persistent loop over the list.
template <typename K, bool kHasValues>
__global__ void __launch_bounds__(MidCfg::kThreads, 4)
    k_local_mid(K* __restrict__ keys, uint32_t* __restrict__ vals, const uint64_t* __restrict__ P16, int R,
                const uint32_t* __restrict__ list, const HeavyCtl* __restrict__ ctl, const MsdPlan* __restrict__ msd) {
  pdl_entry(false);
  if (!__ldg(&msd->use_msd) || __ldg(&msd->rehist)) return;
  const uint32_t nm = __ldg(&ctl->nmid);
  for (uint32_t i = blockIdx.x; i < nm; i += gridDim.x) {
    const uint32_t bkt = __ldg(list + i);
    const uint64_t b0 = __ldg(P16 + bkt);
    const uint32_t m = (uint32_t)(__ldg(P16 + bkt + 1) - b0);
    sort_bin<K, kHasValues, MidCfg>(keys, vals, keys, vals, b0, m, R, (K)((uint64_t)bkt << R));
    __syncthreads();
  }
}


// ---- small inputs (n <= kSmallSortMax): the whole sort in one CTA's shared
// memory — the keys staged once, a stable LSD over the digits that vary on a
// u16 permutation (warp multisplit ranks, as sort_bin's slow path), keys and
// values written through the permutation (values gathered from the input).  Eleven launches of the LSD path cost ~80 us of launch
// latency at 1,000 pairs.
#ifndef FS_SMALL_SORT_MAX
#define FS_SMALL_SORT_MAX 16384
#endif
constexpr int kSmallSortMax = FS_SMALL_SORT_MAX;  // u64 keys: 128 KB + two u16 permutations 64 KB
constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;

template <typename K, bool kHasValues>
struct SmallSmem {
  K keys[kSmallSortMax];
  uint16_t pa[kSmallSortMax], pb[kSmallSortMax];
  uint16_t wh[kSmallWarps][kRadix];
  uint32_t wtot[kSmallWarps];
  unsigned long long or_all, nor_all;
};

template <typename K, bool kHasValues>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_small_sort(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
                 uint32_t* __restrict__ vout, uint32_t n, int key_bits) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<SmallSmem<K, kHasValues>*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) {
    sm.or_all = 0;
    sm.nor_all = 0;
  }
  __syncthreads();
  unsigned long long o = 0, no = 0;
  for (uint32_t i = tid; i < n; i += kSmallThreads) {
    const K k = kin[i];
    sm.keys[i] = k;
    sm.pa[i] = (uint16_t)i;
    o |= k;
    no |= (K)~k;
  }
  o = ((unsigned long long)__reduce_or_sync(kFull, (uint32_t)(o >> 32)) << 32) | __reduce_or_sync(kFull, (uint32_t)o);
  no = ((unsigned long long)__reduce_or_sync(kFull, (uint32_t)(no >> 32)) << 32) | __reduce_or_sync(kFull, (uint32_t)no);
  if (lane == 0) {
    atomicOr(&sm.or_all, o);
    atomicOr(&sm.nor_all, no);
  }
  __syncthreads();
  const unsigned long long mask = key_bits >= 64 ? ~0ull : ((1ull << key_bits) - 1);
  const unsigned long long varying = sm.or_all & sm.nor_all & mask;
  uint16_t* pa = sm.pa;
  uint16_t* pb = sm.pb;
  const uint32_t chunk = ((n + kSmallWarps - 1) / kSmallWarps + 31) & ~31u;
  const uint32_t c0 = min(warp * chunk, n), c1 = min(c0 + chunk, n);
  for (int sh = 0; sh < key_bits; sh += kRadixBits) {
    if (((varying >> sh) & 0xFFu) == 0) continue;  // every key has this digit: the pass is the identity
    for (int i = tid; i < kSmallWarps * kRadix; i += kSmallThreads) (&sm.wh[0][0])[i] = 0;
    __syncthreads();
    uint16_t* whw = sm.wh[warp];
    // pass A: per-warp digit counts over the warp's chunk of the current order
    for (uint32_t j0 = c0; j0 < c1; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool valid = j < c1;
      const uint32_t dg = valid ? (uint32_t)(sm.keys[pa[j]] >> sh) & 0xFFu : 0u;
      const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
      if (valid && lane == 31 - __clz(peers)) whw[dg] = (uint16_t)(whw[dg] + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    // offsets: digit-major, warp-minor (thread d < 256 owns digit d)
    if (tid < kRadix) {
      uint32_t tot = 0;
      for (int w = 0; w < kSmallWarps; ++w) tot += sm.wh[w][tid];
      const uint32_t inc = warp_inclusive_scan<uint32_t>(tot);
      if (lane == 31) sm.wtot[warp] = inc;
    }
    __syncthreads();
    if (tid < kRadix) {
      uint32_t tot = 0;
      for (int w = 0; w < kSmallWarps; ++w) tot += sm.wh[w][tid];
      uint32_t run = warp_inclusive_scan<uint32_t>(tot) - tot;
      for (int w = 0; w < (int)warp; ++w) run += sm.wtot[w];
      for (int w = 0; w < kSmallWarps; ++w) {
        const uint32_t c = sm.wh[w][tid];
        sm.wh[w][tid] = (uint16_t)run;
        run += c;
      }
    }
    __syncthreads();
    // pass B: stable ranks, scatter of the permutation
    for (uint32_t j0 = c0; j0 < c1; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool valid = j < c1;
      const uint16_t p = valid ? pa[j] : (uint16_t)0;
      const uint32_t dg = valid ? (uint32_t)(sm.keys[p] >> sh) & 0xFFu : 0u;
      const uint32_t peers = match_digit8(dg, __ballot_sync(kFull, valid));
      const uint32_t leader = 31 - __clz(peers);
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = whw[dg];
        whw[dg] = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(kFull, old, leader);
      if (valid) pb[old + __popc(peers & lanemask_lt())] = p;
      __syncwarp();
    }
    __syncthreads();
    uint16_t* t = pa;
    pa = pb;
    pb = t;
  }
  for (uint32_t j = tid; j < n; j += kSmallThreads) {
    const uint32_t p = pa[j];
    kout[j] = sm.keys[p];
    if (kHasValues) vout[j] = vin[p];  // inputs and outputs never overlap (ABI)
  }
}

#include "wide_heavy.cuh"
#ifdef FS_LOCAL_PROBE
float g_probe_ms[2];
#endif

// Bins of 2..kTinyMax keys, one warp each (a CTA's barriers and round trips
// would cost more than the sort): every key's rank = #keys of the bin below it
// (ties by arrival), by shuffles; in place (all keys are in registers first).
template <typename K, bool kHasValues>
__global__ void __launch_bounds__(256, 4)
    k_tiny_bins(K* __restrict__ keys, uint32_t* __restrict__ vals, const uint64_t* __restrict__ P16,
                const uint32_t* __restrict__ list, const HeavyCtl* __restrict__ ctl, const MsdPlan* __restrict__ msd) {
  pdl_entry(true);
  constexpr uint32_t kPer = kTinyMax / 32;  // keys per lane
  if (!msd->use_msd || msd->rehist) return;
  const uint32_t nt = ctl->ntiny;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = gridDim.x * (blockDim.x / 32);
  // The next bin's keys are loaded before the current bin is ranked (a warp
  // handles several bins in turn: each would otherwise wait for its loads).
  uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  K k[kPer];
  uint32_t val[kPer];
  uint64_t b0 = 0;
  uint32_t m = 0;
  auto load = [&](uint32_t tt, K (&kk)[kPer], uint32_t (&vv)[kPer], uint64_t& bb, uint32_t& mm) {
    mm = 0;
    if (tt < nt) {
      const uint32_t v = __ldg(list + tt);
      bb = __ldg(P16 + v);
      mm = (uint32_t)(__ldg(P16 + v + 1) - bb);  // 2..kTinyMax, warp-uniform
    }
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t i = q * 32 + lane;
      kk[q] = i < mm ? keys[bb + i] : K(0);
      vv[q] = (kHasValues && i < mm) ? vals[bb + i] : 0u;
    }
  };
  load(t, k, val, b0, m);
  for (; t < nt; t += nw) {
    K kn[kPer];
    uint32_t vn[kPer];
    uint64_t bn = 0;
    uint32_t mn;
    load(t + nw, kn, vn, bn, mn);
    uint32_t r[kPer];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) r[q] = 0;
    if (m <= 32) {  // one key per lane
      for (uint32_t j = 0; j < m; ++j) {
        const K kj = __shfl_sync(kFull, k[0], j);
        r[0] += (kj < k[0]) || (kj == k[0] && j < lane);
      }
    } else {
      for (uint32_t j = 0; j < m; ++j) {
        K kj = 0;
#pragma unroll
        for (uint32_t q = 0; q < kPer; ++q) {
          const K x = __shfl_sync(kFull, k[q], j & 31u);
          if ((j >> 5) == q) kj = x;
        }
#pragma unroll
        for (uint32_t q = 0; q < kPer; ++q) r[q] += (kj < k[q]) || (kj == k[q] && j < q * 32 + lane);
      }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      if (q * 32 + lane < m) {
        keys[b0 + r[q]] = k[q];
        if (kHasValues) vals[b0 + r[q]] = val[q];
      }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      k[q] = kn[q];
      val[q] = vn[q];
    }
    b0 = bn;
    m = mn;
  }
}


// ================================================================ driver
struct WideLayout {
  size_t alt_k = 0, alt_v = 0, partials = 0;
  size_t zero_begin = 0, kbits = 0, spill = 0, l1spill = 0, scan_status = 0, tickets = 0, digit_hist = 0, status = 0,
         zero_end = 0;
  size_t H16 = 0, P16 = 0, vcnt = 0, vbase = 0, lsd = 0, msd = 0, total = 0;
  size_t hctl = 0, hseg0 = 0, hseg1 = 0, hsegl2 = 0, hchunk = 0, hchist = 0, hcbase = 0, hitems = 0;  // k_heavy
  size_t htiny = 0, hbig = 0, hmid = 0;  // bin lists
  uint64_t tiles = 0, status_tiles = 0;
  uint64_t chunk_tiles = 0;  // MSD: tiles per histogram chunk (= level-1 virtual segment)
  int hgrid = 0;             // MSD: histogram CTAs = chunks
  bool use_msd = false;
};

constexpr int kTickets = 16;  // 0..7 LSD passes, 8 MSD level 1, 9 MSD level 2

WideLayout layout(uint64_t n, int key_bytes, int key_bits, bool has_values) {
  WideLayout L;
  const int width = key_bytes * 8;
  if (key_bits <= 0 || key_bits > width) key_bits = width;
  L.use_msd = n >= kMsdMinN && key_bits >= 32;
  L.tiles = (n + kSTile - 1) / kSTile;
  // status words: one row per ticket; level 2 interleaves only if 256 x (most
  // tiles in a segment) fits, level 1 needs chunks x chunk_tiles <= tiles + chunks
  L.status_tiles = L.tiles + (L.use_msd ? L.tiles / 4 + 2 * kSegs : 0);
  const uint64_t sms = (uint64_t)device_info().sm_count;
  L.chunk_tiles = (L.tiles + sms - 1) / sms;  // (>= 16 tiles per chunk at small n: L1 slower, hist no faster)
  L.hgrid = (int)((L.tiles + L.chunk_tiles - 1) / L.chunk_tiles);
  size_t off = 0;
  L.alt_k = off;
  off = align_up(off + (size_t)n * key_bytes);
  L.alt_v = off;
  if (has_values) off = align_up(off + (size_t)n * 4);
  L.partials = off;
  if (L.use_msd) off = align_up(off + (size_t)L.hgrid * kHistWords * 4);
  L.zero_begin = off;  // zeroed by one memset per call
  L.kbits = off;  // OR / OR-of-complement of the non-empty bins, then of the keys (the window)
  if (L.use_msd) off = align_up(off + 5 * sizeof(unsigned long long));  // + the k_keybits done counter
  L.spill = off;
  if (L.use_msd) off = align_up(off + sizeof(unsigned long long) * kHistBins);
  L.l1spill = off;
  if (L.use_msd) off = align_up(off + sizeof(uint32_t) * kRadix * L.hgrid);
  L.scan_status = off;
  if (L.use_msd) off = align_up(off + sizeof(unsigned long long) * (scan_tiles(kHistBins) + 1));
  L.tickets = off;
  off = align_up(off + sizeof(uint32_t) * kTickets);
  L.hctl = off;
  if (L.use_msd) off = align_up(off + sizeof(HeavyCtl));
  L.digit_hist = off;
  off = align_up(off + sizeof(unsigned long long) * kMaxPasses * kRadix);
  L.status = off;
  off = align_up(off + sizeof(unsigned long long) * kRadix * L.status_tiles);
  L.zero_end = off;
  L.H16 = off;
  if (L.use_msd) off = align_up(off + sizeof(uint64_t) * kHistBins);
  L.P16 = off;
  if (L.use_msd) off = align_up(off + sizeof(uint64_t) * (kHistBins + 1));
  L.vcnt = off;
  if (L.use_msd) off = align_up(off + sizeof(uint32_t) * kRadix * L.hgrid);
  L.vbase = off;
  if (L.use_msd) off = align_up(off + sizeof(uint64_t) * kRadix * L.hgrid);
  if (L.use_msd) {
    const HeavyCaps hc = heavy_caps(n);
    L.hseg0 = off;
    off = align_up(off + sizeof(HeavySeg) * hc.segs);
    L.hseg1 = off;
    off = align_up(off + sizeof(HeavySeg) * hc.segs);
    L.hsegl2 = off;
    off = align_up(off + sizeof(HeavySeg) * kSegs);
    L.hchunk = off;
    off = align_up(off + sizeof(uint32_t) * hc.chunks);
    L.hchist = off;
    off = align_up(off + sizeof(uint32_t) * kRadix * hc.chunks);
    L.hcbase = off;
    off = align_up(off + sizeof(uint64_t) * kRadix * hc.chunks);
    L.hitems = off;
    off = align_up(off + sizeof(HeavyItem) * hc.items);
    L.htiny = off;
    off = align_up(off + sizeof(uint32_t) * kHistBins);
    L.hbig = off;
    off = align_up(off + sizeof(uint32_t) * kHistBins);
    L.hmid = off;
    off = align_up(off + sizeof(uint32_t) * kHistBins);
  }
  L.lsd = off;
  off = align_up(off + sizeof(LsdPlan));
  L.msd = off;
  off = align_up(off + sizeof(MsdPlan));
  L.total = off;
  return L;
}

// Launch with programmatic stream serialization (FS_WIDE_PDL); the kernel must
// begin with pdl_entry().
template <typename... Exp, typename... Act>
cudaError_t launch(void (*k)(Exp...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = FS_WIDE_PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...);
}

template <typename K, bool kHasValues>
cudaError_t run(const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, uint64_t n, int key_bits, void* temp,
                cudaStream_t s) {
  const int kb_eff = key_bits <= 0 || key_bits > (int)(8 * sizeof(K)) ? (int)(8 * sizeof(K)) : key_bits;
  if (n <= (uint64_t)kSmallSortMax && (n <= (uint64_t)FS_SMALL_SORT_MSD_MAX || kb_eff < 32)) {
    // one CTA, every pass in shared memory (beyond FS_SMALL_SORT_MSD_MAX keys only where MSD cannot run)
    constexpr int smem = (int)sizeof(SmallSmem<K, kHasValues>);
    cudaError_t e = cudaFuncSetAttribute(k_small_sort<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    phase_event(0, s);
    k_small_sort<K, kHasValues><<<1, kSmallThreads, smem, s>>>(
        kin, vin, kout, vout, (uint32_t)n, kb_eff);
    phase_event(1, s);
    return cudaGetLastError();
  }
  const WideLayout L = layout(n, sizeof(K), key_bits, kHasValues);
  const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
  char* t = (char*)temp;
  K* alt_k = (K*)(t + L.alt_k);
  uint32_t* alt_v = kHasValues ? (uint32_t*)(t + L.alt_v) : nullptr;
  auto* tickets = (uint32_t*)(t + L.tickets);
  auto* dhist = (unsigned long long*)(t + L.digit_hist);
  auto* status = (unsigned long long*)(t + L.status);
  auto* lsd = (LsdPlan*)(t + L.lsd);
  MsdPlan* msd = L.use_msd ? (MsdPlan*)(t + L.msd) : nullptr;
  auto* P16 = (uint64_t*)(t + L.P16);
  const int sms = device_info().sm_count;
  const bool tma = (((uintptr_t)kin | (uintptr_t)kout | (uintptr_t)alt_k) & 15) == 0 &&
                   (!kHasValues || (((uintptr_t)vin | (uintptr_t)vout | (uintptr_t)alt_v) & 15) == 0);

  constexpr int ssmem = (int)sizeof(ScatterSmem<K, kHasValues>);
  cudaError_t e = cudaFuncSetAttribute(k_scatter<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter<K, kHasValues>, kSThreads, ssmem)) !=
      cudaSuccess)
    return e;
  const unsigned sgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * std::max(occ, 1),
                                                                             L.status_tiles));
  ScatterArgs<K> sa{};
  sa.kin = kin; sa.vin = vin; sa.kA = kout; sa.vA = vout; sa.kB = alt_k; sa.vB = alt_v;
  sa.n = n; sa.lsd = lsd; sa.msd = msd; sa.P16 = P16; sa.status = status; sa.tiles = (uint32_t)L.tiles;
  sa.vbase = (const uint64_t*)(t + L.vbase);
  sa.l1_nseg = (uint32_t)L.hgrid;
  sa.l1_chunk_tiles = (uint32_t)L.chunk_tiles;
  sa.tma = tma ? 1 : 0;

  phase_event(0, s);
  // The lookback status words (the bulk of this range: (tiles + tiles/4 + 512) x 2 KB,
  // ~50 us at c5) are zeroed on every call.  Their pass tags keep the passes of one
  // call apart, but the caller's temp may hold anything (the memory-safety tests fill
  // it with random bytes), and a stale or random word carrying the right tag and a
  // set flag would be read as a published prefix; no tag or epoch width makes that
  // impossible, so the zeroing stays.
  if ((e = cudaMemsetAsync(t + L.zero_begin, 0, L.zero_end - L.zero_begin, s)) != cudaSuccess) return e;

  if (L.use_msd) {
    // ---- trie-binned MSD path
    const int top_shift = key_bits - kTopBits;
    auto* partials = (uint32_t*)(t + L.partials);
    auto* spill = (unsigned long long*)(t + L.spill);
    auto* scan_status = (unsigned long long*)(t + L.scan_status);
    auto* H16 = (uint64_t*)(t + L.H16);
    constexpr int hsmem = kHistWords * 4;
    if ((e = cudaFuncSetAttribute(k_top16_hist<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem)) !=
        cudaSuccess)
      return e;
    auto* l1spill = (uint32_t*)(t + L.l1spill);
    auto* vcnt = (uint32_t*)(t + L.vcnt);
    auto* kbits = (unsigned long long*)(t + L.kbits);
    const uint32_t l1w = (uint32_t)(kRadix * L.hgrid);
    if ((e = launch(k_top16_hist<K>, (unsigned)(L.hgrid), 1024, hsmem, s, kin, n, top_shift, L.chunk_tiles * kSTile, partials, spill,
                                                 l1spill, kbits, nullptr)) != cudaSuccess) return e;
    // the window (a common prefix): a decision from the bins, a pass over the
    // keys only if one bin holds them all, and the histogram again only if the
    // window moved (each kernel returns at once otherwise)
    if ((e = launch(k_binbits, (unsigned)(kHistWords / kBinbitsThreads), kBinbitsThreads, 0, s, partials, L.hgrid, kbits,
                                                                        (uint32_t*)(kbits + 4), key_bits, msd,
                                                                        spill, l1spill, l1w)) != cudaSuccess) return e;
    if ((e = launch(k_keybits<K>, ((unsigned)sms), 1024, 0, s, kin, n, kbits + 2, (uint32_t*)(kbits + 4) + 1, key_bits, msd, spill,
                                                l1spill, l1w)) != cudaSuccess) return e;
    if ((e = launch(k_top16_hist<K>, (unsigned)(L.hgrid), 1024, hsmem, s, kin, n, top_shift, L.chunk_tiles * kSTile, partials, spill,
                                                 l1spill, nullptr, msd)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_merge_scan(partials, L.hgrid, spill, nullptr, kHistBins, H16, kHistBins, 0, P16, scan_status,
                               (uint32_t*)(scan_status + scan_tiles(kHistBins)), s)) != cudaSuccess)
      return e;
    auto* hctl = (HeavyCtl*)(t + L.hctl);
    const bool list_big = n < kListBigMaxN;  // one CTA per bin is cheaper once most bins are large
    if ((e = launch(k_bin_lists, (unsigned)(kListGrid), kListThreads, 0, s, H16, P16, n, msd, hctl, (HeavySeg*)(t + L.hseg0),
                                                   (HeavyItem*)(t + L.hitems), (uint32_t*)(t + L.htiny),
                                                   (uint32_t*)(t + L.hmid), (uint32_t*)(t + L.hbig), list_big ? 1 : 0)) != cudaSuccess) return e;
    if ((e = launch(k_msd_plan, (unsigned)(1), kSegs, 0, s, P16, (uint32_t)L.status_tiles, msd, hctl, (HeavySeg*)(t + L.hsegl2))) != cudaSuccess) return e;
    if ((e = launch(k_vseg_counts, (unsigned)(L.hgrid * kVsegSplit), 256, 0, s, partials, l1spill, vcnt, msd)) != cudaSuccess) return e;
    if ((e = launch(k_vseg_scan, (unsigned)(kRadix / 8), 256, 0, s, vcnt, L.hgrid, P16, (uint64_t*)(t + L.vbase), msd)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    phase_event(1, s);
    for (int level = 1; level <= 2; ++level) {
      sa.mode = level;
      sa.pass = 0;
      sa.shift = key_bits - kRadixBits * level;
      sa.ticket = tickets + 7 + level;
      sa.tag = (unsigned long long)(8 + level) << kTagShift;
      if ((e = launch(k_scatter<K, kHasValues>, (unsigned)(sgrid), kSThreads, ssmem, s, sa)) != cudaSuccess) return e;
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      phase_event(1 + level, s);
    }
    // ---- k_heavy: level 2 of uneven buckets, then the recursion into the bins
    //      above the local-sort capacity (returns at once if there is neither)
    HeavyArgs<K> ha{};
    ha.kout = kout; ha.vout = vout; ha.kalt = alt_k; ha.valt = alt_v;
    ha.n = n;
    ha.tma = tma ? 1 : 0;
    ha.ctl = hctl;
    ha.segl2 = (HeavySeg*)(t + L.hsegl2);
    ha.seg0 = (HeavySeg*)(t + L.hseg0);
    ha.seg1 = (HeavySeg*)(t + L.hseg1);
    ha.chunk_seg = (uint32_t*)(t + L.hchunk);
    ha.chist = (uint32_t*)(t + L.hchist);
    ha.cbase = (uint64_t*)(t + L.hcbase);
    ha.items = (HeavyItem*)(t + L.hitems);
    ha.msd = msd;
    constexpr int hvsmem = (int)sizeof(HeavySmem<K, kHasValues>);
    if ((e = cudaFuncSetAttribute(k_heavy<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize, hvsmem)) !=
        cudaSuccess)
      return e;
    int hocc = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hocc, k_heavy<K, kHasValues>, kHeavyThreads, hvsmem)) !=
        cudaSuccess)
      return e;
    if (hocc < 1) return cudaErrorLaunchOutOfResources;
    {  // cooperative launch (every CTA co-resident, so the grid barriers are safe), also PDL
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(hocc * sms));
      cfg.blockDim = dim3(kHeavyThreads);
      cfg.dynamicSmemBytes = (size_t)hvsmem;
      cfg.stream = s;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = FS_WIDE_PDL ? 2 : 1;
      if ((e = cudaLaunchKernelEx(&cfg, k_heavy<K, kHasValues>, ha)) != cudaSuccess) return e;
    }
    phase_event(4, s);
    // ---- per-bin sorts: the 16-bit bins that fit, then the recursion's items
    constexpr int lsmem = LocalSmemLayout::total;
    if ((e = cudaFuncSetAttribute(k_local_sort<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lsmem)) != cudaSuccess)
      return e;
    // small inputs: at most n / 65 bins need a CTA, listed by the plan
    const unsigned lgrid = list_big ? (unsigned)std::min<uint64_t>(kHistBins, n / (kMidCap + 1) + 1)
                                    : (unsigned)kHistBins;
    if ((e = launch(k_local_sort<K, kHasValues>, (unsigned)(lgrid), kLocalThreads, lsmem, s, 
        kout, vout, P16, key_bits - kTopBits, msd, list_big ? (const uint32_t*)(t + L.hbig) : nullptr, hctl)) != cudaSuccess) return e;
    if ((e = launch(k_tiny_bins<K, kHasValues>, ((unsigned)(8 * sms)), 256, 0, s, kout, vout, P16, (const uint32_t*)(t + L.htiny),
                                                                   hctl, msd)) != cudaSuccess) return e;
    constexpr int msmem = LocalLayout<MidCfg>::total;
    if ((e = cudaFuncSetAttribute(k_local_mid<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  msmem)) != cudaSuccess)
      return e;
    const unsigned mgrid = list_big ? (unsigned)std::min<uint64_t>(kHistBins, n / (kTinyMax + 1) + 1)
                                    : (unsigned)(4 * sms);  // large inputs: few mid bins, a persistent loop
    if ((e = launch(k_local_mid<K, kHasValues>, (unsigned)(mgrid), MidCfg::kThreads, msmem, s, kout, vout, P16, key_bits - kTopBits,
                                                                      (const uint32_t*)(t + L.hmid), hctl, msd)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_heavy_items<K, kHasValues>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lsmem)) != cudaSuccess)
      return e;
    if ((e = launch(k_heavy_items<K, kHasValues>, ((unsigned)(2 * sms)), kLocalThreads, lsmem, s, 
        kout, vout, alt_k, alt_v, hctl, (const HeavyItem*)(t + L.hitems), msd)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
#ifdef FS_LOCAL_PROBE
    // Debug probe (scripts/microbench variants only): re-sort the first
    // FS_LOCAL_PROBE bins twice -- cold (evicted since the main launch) and warm
    // (just written, L2-resident) -- and keep both durations.
    if (sizeof(K) == 8 && kHasValues && !list_big) {
      cudaEvent_t ev[3];
      for (auto& x : ev) cudaEventCreate(&x);
      cudaEventRecord(ev[0], s);
      launch(k_local_sort<K, kHasValues>, (unsigned)FS_LOCAL_PROBE, kLocalThreads, lsmem, s, kout, vout, P16,
             key_bits - kTopBits, msd, (const uint32_t*)nullptr, hctl);
      cudaEventRecord(ev[1], s);
      launch(k_local_sort<K, kHasValues>, (unsigned)FS_LOCAL_PROBE, kLocalThreads, lsmem, s, kout, vout, P16,
             key_bits - kTopBits, msd, (const uint32_t*)nullptr, hctl);
      cudaEventRecord(ev[2], s);
      cudaEventSynchronize(ev[2]);
      cudaEventElapsedTime(&g_probe_ms[0], ev[0], ev[1]);
      cudaEventElapsedTime(&g_probe_ms[1], ev[1], ev[2]);
      for (auto& x : ev) cudaEventDestroy(x);
    }
#endif
    phase_event(5, s);
  }

  // ---- LSD path (when MSD was planned: taken only for a common 16-bit prefix; else every kernel returns at once)
  uint64_t hgrid = (n + 511) / 512;
  if (hgrid > (uint64_t)sms * 4) hgrid = (uint64_t)sms * 4;
  if ((e = launch(k_digit_hist<K>, ((unsigned)hgrid), 512, 0, s, kin, n, passes, dhist, msd)) != cudaSuccess) return e;
  if ((e = launch(k_digit_plan, (unsigned)(1), kRadix, 0, s, dhist, n, passes, lsd, msd)) != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int ev0 = L.use_msd ? 6 : 1;
  phase_event(ev0, s);
  for (int p = 0; p < passes; ++p) {
    sa.mode = 0;
    sa.pass = p;
    sa.shift = p * kRadixBits;
    sa.ticket = tickets + p;
    sa.tag = (unsigned long long)(p + 1) << kTagShift;
    if ((e = launch(k_scatter<K, kHasValues>, (unsigned)(sgrid), kSThreads, ssmem, s, sa)) != cudaSuccess) return e;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    phase_event(ev0 + 1 + p, s);
  }
  if ((e = launch(k_copy_if_identity<K, kHasValues>, ((unsigned)(sms * 4)), 256, 0, s, kin, vin, kout, vout, n, lsd, msd)) != cudaSuccess) return e;
  phase_event(ev0 + 1 + passes, s);
  return cudaGetLastError();
}

}  // namespace

size_t wide_temp_bytes(uint64_t n, int key_bytes, int key_bits, bool has_values) {
  return layout(n, key_bytes, key_bits, has_values).total;
}

bool wide_uses_msd(uint64_t n, int key_bytes, int key_bits) {
  return layout(n, key_bytes, key_bits, false).use_msd;
}

cudaError_t wide_sort(const void* keys_in, const uint32_t* vals_in, void* keys_out, uint32_t* vals_out, uint64_t n,
                      int key_bytes, int key_bits, void* temp, size_t temp_bytes, cudaStream_t s) {
  (void)temp_bytes;
  if (key_bytes == 4)
    return run<uint32_t, false>((const uint32_t*)keys_in, nullptr, (uint32_t*)keys_out, nullptr, n, key_bits, temp, s);
  if (vals_in)
    return run<uint64_t, true>((const uint64_t*)keys_in, vals_in, (uint64_t*)keys_out, vals_out, n, key_bits, temp,
                               s);
  return run<uint64_t, false>((const uint64_t*)keys_in, nullptr, (uint64_t*)keys_out, nullptr, n, key_bits, temp, s);
}

}  // namespace fs

#ifdef FS_LOCAL_PROBE
extern "C" void fs_probe_local_ms(float* out) { out[0] = fs::g_probe_ms[0]; out[1] = fs::g_probe_ms[1]; }
#endif
