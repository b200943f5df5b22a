// hist16.cu — stages 1 and 2 of the u16 path (G1 + G2): the per-SM compressed
// histogram, the merge of the per-SM histograms, and the exclusive scan, in one
// cooperative kernel.
//
// What it computes (§III.B.1 Fractal RMW, Alg. 1):
// every key increments the counter of the leaf its MSB-first bit path selects;
// at p = 16 the leaf slot is the key itself (ledger 1; computable pointers,
// PAPER.md:196-215).  The trie's internal levels are sums of leaves (SIBLING
// SUM), so only the leaf level is materialised; the scan builds
// the rest implicitly.  Then C[v] = sum over SMs (the two-step
// local -> global merge) and P[v] = sum_{u<v} C[u] =
// GetIndex(v) for every v (Alg. 3).
//
// B200 design:
//  * Cooperative launch, one CTA of 1024 threads per SM.  The 65,536-bin local
//    tree lives in shared memory as 16-bit counters packed two per 32-bit word
//    (128 KB): counter-width tapering (§III.D.1) is what makes a
//    privatised 65,536-bin histogram fit in one SM (n_L = W/w_c = 2 counters
//    per word).  Bin v lives in word v>>1, half v&1, so a packed
//    partial is exactly a u16 array indexed by bin.
//  * Keys stream in as 128-bit evict-first loads, two vectors (16 keys) per
//    thread per group.  The loop is bound by the shared-memory atomic unit
//    (~3.5 wavefronts per warp-wide random atomic from bank conflicts); the
//    micro-benchmarks behind these choices are in DESIGN.md §Kernels/hist16.
//  * Overflow ("Counter Width Compression and Overflow", ledger 12):
//    never wraps.  Every shared atomic returns the old word; the returns of a
//    group are OR-ed and tested once.  If either half of any returned word was
//    >= THETA = 2^15, the thread re-reads each word it touched and atomically
//    exchanges every word that is still hot with 0, adding both halves to the
//    global u64 spill array.  Between the increment that lifts a counter to
//    >= THETA and the first exchange, each thread adds at most one group (16
//    keys) to it, because it tests before its next group; so a counter never
//    exceeds THETA + 255 + 1024 * 16 = 49,407 < 65,536.  No barrier is needed.
//  * Runs of equal keys (sorted or constant inputs, ledger 21-22): a warp that
//    sees an all-equal vector switches to an aggregating mode (one +8 per
//    thread or one +256 per warp instead of same-address atomics); the check is
//    sampled every 4th group while not aggregating.  Vectors with mixed keys
//    are queued per warp and counted 32 at a time by a full-warp add8.
//  * Prologue zeroes the spill array (grid-strided) and the grid synchronises
//    once, so the call needs no memset node.
//  * Tail: each CTA flushes its partial (L2-resident), grid sync, then 128
//    slices of 512 bins are merged (16 row groups x 64 columns of 16-byte
//    loads).  For the sort, each slice writes its local exclusive prefix and
//    its total; the 128-entry scan of the totals is done by the expansion
//    kernel's first search round (no cross-slice pass here).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

#ifdef FS_HIST_TRACE
// Debug-only phase timestamps (scripts/microbench/hist_trace.cu builds this file
// with -DFS_HIST_TRACE); compiled out of libfractalsort.so.
__device__ unsigned long long g_hist_trace[256][8];
#define FS_TRACE(i)                                                                    \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      unsigned long long t_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      g_hist_trace[blockIdx.x][i] = t_;                                                \
      unsigned smid_;                                                                  \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                               \
      g_hist_trace[blockIdx.x][7] = smid_;                                             \
    }                                                                                  \
  } while (0)
#else
#define FS_TRACE(i) \
  do {              \
  } while (0)
#endif

namespace fs {
namespace {

constexpr int kThreads = 1024;
constexpr int kUnroll = 2;                  // 128-bit vectors per thread per group
constexpr uint32_t kHotMask = 0x80008000u;  // either 16-bit half >= 2^15
constexpr int kMaxGrid = 1024;              // CTAs (one per SM): the merge loops over rows
constexpr int kSmallGrid = 32;              // up to this many CTAs, the merge of stage 1b is column-per-thread
static_assert(32768 + 255 + kThreads * kUnroll * 8 < 65536, "spill bound violated");

#ifndef FS_HIST_HOT
#define FS_HIST_HOT 1
#endif
#ifndef FS_HIST_HOT_ALWAYS
#define FS_HIST_HOT_ALWAYS 0
#endif
// The CTA's hot key (skewed inputs): the first key whose counter crossed 2^15
// (0xFFFFFFFF: none yet).  Warps that see it count that key in registers.
__shared__ uint32_t s_hot_key;
// (A third hot word, redirected the same way, measured slower on Zipf: 258.6 ->
// 283.1 us, 280.2 with FS_HIST_FMA 2; profiles/r02g/u16_variants_hot3.txt.)
// FS_HIST_HOT2W: a second hot word (the first spill of another word once the
// first is set), redirected to a second per-thread dummy.
#ifndef FS_HIST_HOT2W
#define FS_HIST_HOT2W 1
#endif
__shared__ uint32_t s_hot_key2;

FS_DEVINL void spill_word(uint32_t* sh, uint32_t w, unsigned long long* spill) {
  const uint32_t x = atomicExch(&sh[w], 0u);
  if (FS_HIST_HOT) {
    const uint32_t k = (x & 0xFFFFu) >= (x >> 16) ? 2 * w : 2 * w + 1;
    const uint32_t prev = atomicCAS(&s_hot_key, 0xFFFFFFFFu, k);
    if (FS_HIST_HOT2W && prev != 0xFFFFFFFFu && (prev >> 1) != w) atomicCAS(&s_hot_key2, 0xFFFFFFFFu, k);
  }
  if (x & 0xFFFFu) atomicAdd(&spill[2 * w], (unsigned long long)(x & 0xFFFFu));
  if (x >> 16) atomicAdd(&spill[2 * w + 1], (unsigned long long)(x >> 16));
}

// Add `cnt` (<= 256) to bin k; spill if the counter word was hot.
FS_DEVINL void add_key(uint32_t* sh, uint32_t k, uint32_t cnt, unsigned long long* spill) {
  const uint32_t w = k >> 1;
  const uint32_t old = atomicAdd(&sh[w], (k & 1u) ? (cnt << 16) : cnt);
  if (old & kHotMask) spill_word(sh, w, spill);
}

// FS_HIST_FMA: the increments and the high key's shift computed on the FMA pipe
// (IMAD / IMAD.HI) instead of the ALU pipe.  The ALU pipe is what saturates in
// the redirecting (skewed-input) loop: its two compare + select pairs per key
// come on top of the plain loop's address and increment arithmetic, and the
// compiler turns (b * 0xFFFF + 1) into compare + select and max(.., 1) into
// VIMNMX, all ALU (profiles/ncu_summary_r02f_c3a.md: math_pipe_throttle).
// Zipf 265.7 -> 258.5 us per sort, other inputs unchanged; moving the masks
// and bit extractions over as well (ALU:FMA 74:65 instead of 103:38 in the
// redirecting block) gained nothing more (profiles/r02g/u16_variants_fma.txt).
#ifndef FS_HIST_FMA
#define FS_HIST_FMA 1
#endif
// b * 0xFFFF + 1 for a bit b: 1 or 0x10000 (one IMAD; opaque to the compiler's select rewrite)
FS_DEVINL uint32_t inc_of_bit(uint32_t b) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, 65535, 1;" : "=r"(r) : "r"(b));
  return r;
}
// x >> k as the high word of x * 2^(32 - k) (IMAD.HI)
template <int k>
FS_DEVINL uint32_t shr_hi(uint32_t x) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(1u << (32 - k)));
  return r;
}
// Word byte offset and increment of the low / high key of a packed pair x.
FS_DEVINL uint32_t addr_lo(uint32_t x) { return (x + x) & 0x1FFFCu; }
FS_DEVINL uint32_t addr_hi(uint32_t x) { return (FS_HIST_FMA ? shr_hi<15>(x) : (x >> 15)) & 0x1FFFCu; }
FS_DEVINL uint32_t inc_lo(uint32_t x) { return FS_HIST_FMA ? inc_of_bit(x & 1u) : (x & 1u) * 0xFFFFu + 1u; }
FS_DEVINL uint32_t inc_hi(uint32_t x) { return FS_HIST_FMA ? inc_of_bit(shr_hi<16>(x) & 1u) : max(x & 0x10000u, 1u); }

// 8 atomics; returns the OR of the old words.  Word byte offset of the low key
// of x is (x & 0xFFFE) * 2, of the high key (x >> 17) * 4; the increment is 1 or
// 0x10000 by the key's lowest bit.
FS_DEVINL uint32_t add8(uint32_t* sh, const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  char* base = reinterpret_cast<char*>(sh);
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + addr_lo(x)), inc_lo(x));
    acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + addr_hi(x)), inc_hi(x));
  }
  return acc;
}

// add8 for skewed inputs: keys equal to the hot key `h` are counted in a
// register (hc) instead of contending for one shared-memory word.
// FS_HIST_REDIRECT: branch-free -- every key still issues its atomic, but a hot
// key's goes to this thread's private dummy word (dummy_off, bank = lane, always
// 0) with increment 0, so a warp instruction never serialises on the hot word
// and no branch splits the warp (round 1 branched around the atomic: 2.4x the
// instructions of the uniform loop, profiles/r02/ncu_hist_skew.md).
#ifndef FS_HIST_REDIRECT
#define FS_HIST_REDIRECT 1
#endif
// FS_HIST_HOTWORD: h is the hot key's word byte offset, the dummy counts both of
// its keys (see below); folded into the spill by hot_dummy_flush.
#ifndef FS_HIST_HOTWORD
#define FS_HIST_HOTWORD 1
#endif
FS_DEVINL uint32_t add8_hot(uint32_t* sh, const uint4& v, uint32_t h, uint32_t& hc, uint32_t dummy_off,
                            uint32_t h2 = 0xFFFFFFFFu, uint32_t dummy2_off = 0) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  char* base = reinterpret_cast<char*>(sh);
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t x = w[j];
    if (FS_HIST_HOTWORD) {
      // the hot key's whole counter WORD goes to the dummy with the normal
      // increment: the dummy's halves count keys 2w and 2w + 1 exactly as the
      // table's word would, so one word compare replaces key extraction,
      // compare, increment select and register count.
      const uint32_t a0 = addr_lo(x), a1 = addr_hi(x);
      uint32_t b0 = a0 == h ? dummy_off : a0, b1 = a1 == h ? dummy_off : a1;
      if (FS_HIST_HOT2W) {
        b0 = a0 == h2 ? dummy2_off : b0;
        b1 = a1 == h2 ? dummy2_off : b1;
      }
      acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + b0), inc_lo(x));
      acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + b1), inc_hi(x));
    } else if (FS_HIST_REDIRECT) {
      const bool pl = (x & 0xFFFFu) == h, ph = (x >> 16) == h;
      hc += (uint32_t)pl + (uint32_t)ph;
      acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + (pl ? dummy_off : ((x + x) & 0x1FFFCu))),
                       pl ? 0u : (x & 1u) * 0xFFFFu + 1u);
      acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + (ph ? dummy_off : ((x >> 15) & 0x1FFFCu))),
                       ph ? 0u : max(x & 0x10000u, 1u));
    } else {
      if ((x & 0xFFFFu) != h) acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + ((x + x) & 0x1FFFCu)), (x & 1u) * 0xFFFFu + 1u);
      else ++hc;
      if ((x >> 16) != h) acc |= atomicAdd(reinterpret_cast<uint32_t*>(base + ((x >> 15) & 0x1FFFCu)), max(x & 0x10000u, 1u));
      else ++hc;
    }
  }
  return acc;
}

// Slow path after a hot return: exchange every touched word that is still hot.
FS_DEVINL void recheck8(uint32_t* sh, const uint4& v, unsigned long long* spill) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = (w[j] & 0xFFFFu) >> 1, b = w[j] >> 17;
    if (sh[a] & kHotMask) spill_word(sh, a, spill);
    if (sh[b] & kHotMask) spill_word(sh, b, spill);
  }
}

// FS_HIST_HOTWORD: move the dummy word's two halves (the hot word's keys 2w,
// 2w + 1 counted by this thread) into the spill.  `force`: at the end; else only
// once a half reached 2^15 (the dummy obeys the same bound as any table word).
FS_DEVINL void hot_dummy_flush(uint32_t* sh, uint32_t dummy_off, uint32_t hot_key, unsigned long long* spill,
                               bool force) {
  uint32_t* d = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(sh) + dummy_off);
  if (!force && !(*d & kHotMask)) return;
  const uint32_t x = atomicExch(d, 0u);
  const uint32_t k0 = hot_key & ~1u;
  if (x & 0xFFFFu) atomicAdd(&spill[k0], (unsigned long long)(x & 0xFFFFu));
  if (x >> 16) atomicAdd(&spill[k0 + 1], (unsigned long long)(x >> 16));
}

FS_DEVINL bool all8_equal(const uint4& v) {
  return (v.x == v.y) & (v.y == v.z) & (v.z == v.w) & ((v.x >> 16) == (v.x & 0xFFFFu));
}

// Aggregating path for a vector when the warp has runs of equal keys (sorted or
// constant inputs).  Lanes whose 8 keys all equal lane 0's key ka (or lane 31's
// kb: a run boundary inside the warp) are counted by one atomic of
// 8 * (number of such lanes) <= 256; other all-equal lanes add 8; a lane with
// mixed keys (a run boundary or an outlier of a nearly sorted input) takes the
// plain path.  (Taking its keys equal to ka / kb out of the atomics -- the
// hot-key redirect -- cut c3c's atomic wavefronts from 37.3 M to 16.6 M but the
// divergent lanes' extra instructions made the loop issue-bound: 286 -> 384 us,
// 334 us with ka alone; a warp-wide __reduce_add_sync of the run counts: constant
// keys 192 -> 277 us.  profiles/r02/u16_variants_redirect.txt,
// u16_variants_agg_redirect_lean.txt.)
#ifndef FS_HIST_MIXQ
#define FS_HIST_MIXQ 1
#endif
// Per-warp queue of mixed vectors (FS_HIST_MIXQ): 64 uint4 slots in shared
// memory after the dummy words, a ring read 32 at a time.
constexpr int kMixQ = 64;
struct MixQ {
  uint4* q;      // this warp's ring
  uint32_t h, n;  // head, entries (warp-uniform)
};

// Count the queued vectors [h, h + cnt) with one full-warp add8 (lane l takes slot h + l).
FS_DEVINL void mixq_drain(uint32_t* sh, MixQ& mq, uint32_t cnt, unsigned long long* spill) {
  __syncwarp();
  const uint32_t lane = lane_id();
  if (lane < cnt) {
    const uint4 w = mq.q[(mq.h + lane) & (kMixQ - 1)];
    if (add8(sh, w) & kHotMask) recheck8(sh, w, spill);
  }
  __syncwarp();  // the slots just read may be refilled by the next enqueue
  mq.h = (mq.h + cnt) & (kMixQ - 1);
  mq.n -= cnt;
}

FS_DEVINL void add8_agg(uint32_t* sh, const uint4& v, unsigned long long* spill, MixQ& mq) {
  const uint32_t lane = lane_id();
  const bool eq = all8_equal(v);
  const uint32_t k0 = v.x & 0xFFFFu;
  const uint32_t ka = __shfl_sync(kFull, k0, 0), kb = __shfl_sync(kFull, k0, 31);  // all lanes shuffle
  const uint32_t ma = __ballot_sync(kFull, eq && k0 == ka);
  const uint32_t mb = __ballot_sync(kFull, eq && k0 == kb && k0 != ka);
  if (lane == 0 && ma) add_key(sh, ka, 8u * __popc(ma), spill);
  if (lane == 31 && mb) add_key(sh, kb, 8u * __popc(mb), spill);
  const bool in = ((ma | mb) >> lane) & 1u;
#if FS_HIST_MIXQ
  // A lane with mixed keys (a run boundary, or an outlier of a nearly sorted
  // input: ~8% of c3c's vectors) is queued instead of issuing 8 atomics with
  // the warp's other lanes idle; every 32 queued vectors are counted by one
  // full-warp add8 (then checked, so the spill bound is unchanged: a thread
  // adds at most 8 keys before its check).
  if ((ma | mb) == kFull) return;  // warp-uniform: the whole warp is one or two runs (constant keys)
  if (!in && eq) add_key(sh, k0, 8u, spill);
  const bool mixed = !in && !eq;
  const uint32_t mm = __ballot_sync(kFull, mixed);
  if (mm) {  // warp-uniform
    if (mixed) mq.q[(mq.h + mq.n + __popc(mm & lanemask_lt())) & (kMixQ - 1)] = v;
    mq.n += __popc(mm);
    if (mq.n >= 32) mixq_drain(sh, mq, 32, spill);
  }
#else
  if (in) return;
  if (eq) {
    add_key(sh, k0, 8u, spill);
    return;
  }
  if (add8(sh, v) & kHotMask) recheck8(sh, v, spill);
#endif
}

constexpr int kSliceBins = 512;                    // merge/scan granularity
constexpr int kSlices = kHistBins / kSliceBins;    // 128
constexpr int kSliceVec = kSliceBins / 8;          // uint4 per partial row per slice (64)
constexpr int kRowGroups = kThreads / kSliceVec;   // 16
static_assert(kSlices == kHistSlices, "slice count");

struct HistArgs {
  const uint16_t* keys;
  uint64_t n, head, nvec;
  uint32_t* partials;                  // grid x kHistWords packed u16 pairs
  unsigned long long* spill;           // 65536 u64 (zeroed in the prologue)
  uint64_t* hist_out;                  // optional: C written (+=) for v < nbins_out
  uint64_t nbins_out;
  int accumulate;
  uint64_t* prefix;                    // optional: slice-local exclusive prefix L[65536] (the sort path)
  uint64_t* slice_tot;                 // with prefix: the 128 slice totals
};

__global__ void __launch_bounds__(kThreads, 1) k_hist16(HistArgs a) {
  extern __shared__ uint4 smem_v4[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem_v4);
  const uint32_t tid = threadIdx.x;
  cg::grid_group grid = cg::this_grid();
  FS_TRACE(0);

  // ---------------- prologue: zero the local tree, the spill array and the flags
#pragma unroll
  for (int i = 0; i < kHistWords / 4 / kThreads; ++i) smem_v4[tid + i * kThreads] = make_uint4(0, 0, 0, 0);
  sh[kHistWords + tid] = 0;  // dummy words (FS_HIST_REDIRECT)
  for (uint32_t i = blockIdx.x * kThreads + tid; i < kHistBins + 1; i += gridDim.x * kThreads) a.spill[i] = 0;
  if (tid == 0) s_hot_key = s_hot_key2 = 0xFFFFFFFFu;
  if (FS_HIST_HOT2W) sh[kHistWords + kThreads + (FS_HIST_MIXQ ? kThreads / 32 * kMixQ * 4 : 0) + tid] = 0;
  grid.sync();
  FS_TRACE(1);

  // ---------------- stage 1: local compressed histogram
  // Unaligned head and ragged tail (< 8 + 7 keys) go to the last CTA, one key per thread.
  if (blockIdx.x == gridDim.x - 1) {
    const uint64_t tail0 = a.head + a.nvec * 8;
    const uint64_t nscalar = a.head + (a.n - tail0);
    for (uint64_t t = tid; t < nscalar; t += kThreads) {
      const uint64_t idx = t < a.head ? t : tail0 + (t - a.head);
      add_key(sh, a.keys[idx], 1u, a.spill);
    }
  }
  const uint4* __restrict__ vec = reinterpret_cast<const uint4*>(a.keys + a.head);
  const uint64_t nvec = a.nvec;
  // Work is split into groups of kUnroll x 1024 vectors (16,384 keys).  Most
  // groups are assigned statically (grid-strided); the last 1/16 are handed out
  // dynamically in warp-sized chunks (2,048 keys) from a global counter,
  // because SMs run the atomic-bound loop at rates ~8% apart (hist_trace:
  // per-CTA loop 115-125 us on 2^28 keys).  Per-warp tickets need no CTA
  // barrier, so no warp waits on another's loads.
  constexpr uint64_t kGroupVec = (uint64_t)kUnroll * kThreads;
#ifndef FS_HIST_CHUNK_ITERS  // scripts/microbench sweeps
#define FS_HIST_CHUNK_ITERS 4
#endif
#ifndef FS_HIST_DYN_DIV
#define FS_HIST_DYN_DIV 16
#endif
  constexpr int kChunkIters = FS_HIST_CHUNK_ITERS;
  constexpr uint64_t kChunkVec = (uint64_t)kChunkIters * kUnroll * 32;
  static_assert(kGroupVec % kChunkVec == 0, "chunks tile the groups");
  const uint64_t ngroups = nvec / kGroupVec;
  const uint64_t nstatic = ngroups - ngroups / FS_HIST_DYN_DIV;
  bool agg = false;
  uint32_t phase = 0;
  const uint32_t dummy_off = (kHistWords + tid) * 4u;  // this thread's dummy word (bank = lane, stays 0)
  uint32_t hot = 0xFFFFFFFFu, hot_cnt = 0;  // this warp's view of s_hot_key, refreshed every 4th group
  uint32_t hot2 = 0xFFFFFFFFu;
  const uint32_t dummy2_off = (kHistWords + kThreads + (FS_HIST_MIXQ ? kThreads / 32 * kMixQ * 4 : 0) + tid) * 4u;
  MixQ mq{reinterpret_cast<uint4*>(sh + kHistWords + kThreads) + (tid >> 5) * kMixQ, 0u, 0u};
  // the whole warp calls this together (warp votes inside)
  auto process_v = [&](uint4 (&v)[kUnroll]) {
    if (agg || phase == 0) {
      if (FS_HIST_HOT) hot = s_hot_key;  // one broadcast load: warp-uniform
      if (FS_HIST_HOT2W) hot2 = s_hot_key2;
      bool runs = false;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) runs |= all8_equal(v[u]);
      agg = __any_sync(kFull, runs);
    }
    phase = (phase + 1) & 3;
    if (agg) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) add8_agg(sh, v[u], a.spill, mq);
    } else {
      uint32_t acc = 0;
      if (FS_HIST_HOT && (FS_HIST_HOT_ALWAYS || hot != 0xFFFFFFFFu)) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          acc |= add8_hot(sh, v[u], FS_HIST_HOTWORD ? (hot >> 1) * 4u : hot, hot_cnt, dummy_off, (hot2 >> 1) * 4u,
                          dummy2_off);
        if (FS_HIST_HOTWORD && (acc & kHotMask)) {
          hot_dummy_flush(sh, dummy_off, hot, a.spill, false);
          if (FS_HIST_HOT2W && hot2 != 0xFFFFFFFFu) hot_dummy_flush(sh, dummy2_off, hot2, a.spill, false);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) acc |= add8(sh, v[u]);
      }
      if (acc & kHotMask) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) recheck8(sh, v[u], a.spill);
      }
    }
  };
  // Static groups, software-pipelined: group g + G is loaded before group g's
  // atomics, so a warp never waits on HBM between its atomic bursts
  // (c2: 225.7 -> 221.8 us per sort).
  if (blockIdx.x < nstatic) {
    uint4 cur[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) cur[u] = ld_stream_v4(vec + blockIdx.x * kGroupVec + u * kThreads + tid);
    for (uint64_t g = blockIdx.x; g < nstatic; g += gridDim.x) {
      uint4 nxt[kUnroll];
      const bool more = g + gridDim.x < nstatic;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        nxt[u] = more ? ld_stream_v4(vec + (g + gridDim.x) * kGroupVec + u * kThreads + tid) : make_uint4(0, 0, 0, 0);
      process_v(cur);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) cur[u] = nxt[u];
    }
  }
  FS_TRACE(6);  // (debug trace: thread 0's static groups done)
  {
    unsigned int* work = reinterpret_cast<unsigned int*>(a.spill + kHistBins);
    const uint64_t dyn0 = nstatic * kGroupVec;
    const uint64_t nchunks = (ngroups * kGroupVec - dyn0) / kChunkVec;
    const uint32_t lane = lane_id();
    for (;;) {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(work, 1u);
      c = __shfl_sync(kFull, c, 0);
      if (c >= nchunks) break;
      const uint4* p = vec + dyn0 + (uint64_t)c * kChunkVec + lane;
      uint4 cur[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) cur[u] = ld_stream_v4(p + u * 32);
#pragma unroll 1
      for (int j = 0; j < kChunkIters; ++j) {  // pipelined like the static loop
        uint4 nxt[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          nxt[u] = j + 1 < kChunkIters ? ld_stream_v4(p + (j + 1) * kUnroll * 32 + u * 32) : make_uint4(0, 0, 0, 0);
        process_v(cur);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) cur[u] = nxt[u];
      }
    }
  }
  if (FS_HIST_MIXQ && mq.n) mixq_drain(sh, mq, mq.n, a.spill);  // the warp's last queued vectors
  if (FS_HIST_HOT && FS_HIST_HOTWORD && hot != 0xFFFFFFFFu) {
    // this thread's dummy: the hot word's two counters -> warp sums -> the global spill once
    const uint32_t x = sh[kHistWords + tid];
    const uint32_t lo = warp_sum(x & 0xFFFFu), hi = warp_sum(x >> 16);
    if (lane_id() == 0) {
      if (lo) atomicAdd(&a.spill[hot & ~1u], (unsigned long long)lo);
      if (hi) atomicAdd(&a.spill[hot | 1u], (unsigned long long)hi);
    }
  }
  if (FS_HIST_HOT2W && hot2 != 0xFFFFFFFFu) {
    const uint32_t x = sh[dummy2_off / 4];
    const uint32_t lo = warp_sum(x & 0xFFFFu), hi = warp_sum(x >> 16);
    if (lane_id() == 0) {
      if (lo) atomicAdd(&a.spill[hot2 & ~1u], (unsigned long long)lo);
      if (hi) atomicAdd(&a.spill[hot2 | 1u], (unsigned long long)hi);
    }
  }
  if (FS_HIST_HOT && !FS_HIST_HOTWORD && hot != 0xFFFFFFFFu) {  // keys counted in registers: added to the global spill once
    const uint32_t t = warp_sum(hot_cnt);
    if (lane_id() == 0 && t) atomicAdd(&a.spill[hot], (unsigned long long)t);
  }
  // Vectors after the last full group (< 2,048).
  for (uint64_t i = ngroups * kGroupVec + (uint64_t)blockIdx.x * kThreads + tid; i < nvec;
       i += (uint64_t)gridDim.x * kThreads) {
    const uint4 q = ld_stream_v4(vec + i);
    if (add8(sh, q) & kHotMask) recheck8(sh, q, a.spill);
  }
  __syncthreads();
  FS_TRACE(2);

  // Flush the local tree: the first step of the two-step merge.
  uint4* dst = reinterpret_cast<uint4*>(a.partials + (uint64_t)blockIdx.x * kHistWords);
#ifndef FS_HIST_TMA_FLUSH
#define FS_HIST_TMA_FLUSH 1
#endif
  if (FS_HIST_TMA_FLUSH) {
    // 8 bulk copies of 16 KB (cp.async.bulk, the TMA engine) instead of 32 K
    // thread stores: the table was written by every thread's atomics (generic
    // proxy), so all threads fence towards the async proxy before the barrier.
    fence_proxy_async_smem();
    __syncthreads();
    constexpr uint32_t kPiece = kHistWords * 4 / 8;
    if (tid < 8) {
      bulk_s2g(reinterpret_cast<char*>(dst) + tid * kPiece, reinterpret_cast<char*>(sh) + tid * kPiece, kPiece);
      bulk_commit();
      bulk_wait_all();
    }
  } else {
#pragma unroll
    for (int j = 0; j < kHistWords / 4 / kThreads; ++j) dst[tid + j * kThreads] = smem_v4[tid + j * kThreads];
  }
  FS_TRACE(3);
  grid.sync();
  FS_TRACE(4);
  // The dependent kernel (expansion) may start launching; it waits for this
  // grid's completion before reading P (programmatic dependent launch).
  cudaTriggerProgrammaticLaunchCompletion();

  // ---------------- stage 1b: merge
  const int G = gridDim.x;
  if (G <= kSmallGrid) {
    // Few CTAs (small n): each thread owns one 8-bin column of one of this
    // CTA's slices and sums all G rows itself; a slice's 64 columns are two
    // warps, which scan their 512 bins together.  16 slices per round.
    __shared__ unsigned long long pair_tot[kThreads / 32];
    const uint32_t my_slices = (kSlices - blockIdx.x + G - 1) / G;
    constexpr uint32_t kPerRound = kThreads / kSliceVec;  // 16
    for (uint32_t r0 = 0; r0 < my_slices; r0 += kPerRound) {
      const uint32_t s_local = r0 + tid / kSliceVec, c = tid % kSliceVec;
      const bool active = s_local < my_slices;
      const uint32_t slice = blockIdx.x + s_local * G;
      uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (active) {
        const uint4* src = reinterpret_cast<const uint4*>(a.partials) + (uint64_t)slice * kSliceVec + c;
#pragma unroll 4
        for (int g = 0; g < G; ++g) {
          const uint4 q = __ldcg(src + (uint64_t)g * (kHistWords / 4));
          acc[0] += q.x & 0xFFFFu; acc[1] += q.x >> 16; acc[2] += q.y & 0xFFFFu; acc[3] += q.y >> 16;
          acc[4] += q.z & 0xFFFFu; acc[5] += q.z >> 16; acc[6] += q.w & 0xFFFFu; acc[7] += q.w >> 16;
        }
      }
      unsigned long long cnt[8], tot = 0;
      const uint32_t bin0 = slice * kSliceBins + c * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = active ? acc[j] + a.spill[bin0 + j] : 0ull;
        tot += cnt[j];
        if (active && a.hist_out && bin0 + j < a.nbins_out)
          a.hist_out[bin0 + j] = a.accumulate ? a.hist_out[bin0 + j] + cnt[j] : cnt[j];
      }
      if (a.prefix) {
        // exclusive scan over the slice's 64 columns (warps 2k and 2k+1)
        const unsigned long long inc = warp_inclusive_scan<unsigned long long>(tot);
        if ((tid & 31) == 31) pair_tot[tid >> 5] = inc;
        __syncthreads();
        unsigned long long run = inc - tot + (((tid >> 5) & 1) ? pair_tot[(tid >> 5) - 1] : 0ull);
        if (active) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            a.prefix[bin0 + j] = run;
            run += cnt[j];
          }
          if (c == kSliceVec - 1) a.slice_tot[slice] = run;
        }
        __syncthreads();  // pair_tot is reused by the next round
      }
    }
    FS_TRACE(5);
    return;
  }
  uint32_t* part = sh;                                                                       // [16][512] u32
  unsigned long long* wsum = reinterpret_cast<unsigned long long*>(sh + kRowGroups * kSliceBins);  // [16]
  const uint32_t col = tid % kSliceVec, rg = tid / kSliceVec;
  for (int slice = blockIdx.x; slice < kSlices; slice += G) {
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint4* src = reinterpret_cast<const uint4*>(a.partials) + (uint64_t)slice * kSliceVec + col;
    // the spill of this thread's bin, fetched together with the partial rows
    const unsigned long long spilled = tid < kSliceBins ? __ldcg(a.spill + slice * kSliceBins + tid) : 0ull;
    // All of this thread's rows (G <= 160: one batch) are loaded before any is
    // summed, so the merge costs one L2 round trip instead of ceil(G / 64).
    constexpr int kBatch = 10;
    for (int g0 = rg; g0 < G; g0 += kBatch * kRowGroups) {
      uint4 q[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int g = g0 + u * kRowGroups;
        q[u] = g < G ? __ldcg(src + (uint64_t)g * (kHistWords / 4)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        acc[0] += q[u].x & 0xFFFFu; acc[1] += q[u].x >> 16; acc[2] += q[u].y & 0xFFFFu; acc[3] += q[u].y >> 16;
        acc[4] += q[u].z & 0xFFFFu; acc[5] += q[u].z >> 16; acc[6] += q[u].w & 0xFFFFu; acc[7] += q[u].w >> 16;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) part[rg * kSliceBins + col * 8 + j] = acc[j];
    __syncthreads();
    unsigned long long c = 0;
    const uint32_t bin = slice * kSliceBins + tid;
    if (tid < kSliceBins) {
#pragma unroll
      for (int r = 0; r < kRowGroups; ++r) c += part[r * kSliceBins + tid];
      c += spilled;
      if (a.hist_out && bin < a.nbins_out) a.hist_out[bin] = a.accumulate ? a.hist_out[bin] + c : c;
    }
    if (a.prefix) {
      // slice-local exclusive scan L[v] and the slice total; the expansion
      // kernel adds the slice bases (two-level prefix, see expand16.cu)
      const unsigned long long inc = warp_inclusive_scan<unsigned long long>(c);
      if ((tid & 31) == 31 && tid < kSliceBins) wsum[tid >> 5] = inc;
      __syncthreads();
      unsigned long long off = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kSliceBins / 32; ++w) {
        const unsigned long long t = wsum[w];
        if (w < (int)(tid >> 5)) off += t;
        tot += t;
      }
      if (tid < kSliceBins) a.prefix[bin] = off + inc - c;
      if (tid == 0) a.slice_tot[slice] = tot;
    }
    __syncthreads();
  }
  FS_TRACE(5);
}

}  // namespace

int hist16_grid(uint64_t n) {
#ifndef FS_HIST_KEYS_PER_CTA
#define FS_HIST_KEYS_PER_CTA 8192
#endif
  // keep >= FS_HIST_KEYS_PER_CTA keys per CTA: every CTA zeroes and flushes 128 KB,
  // but below ~2^24 keys the loop is short and more CTAs win (u16 sort b2b,
  // 65,536 -> 8,192 keys per CTA: 2^20 26.8 -> 23.0 us, 2^22 33.0 -> 29.1 us,
  // 2^24 unchanged; profiles/r02d/u16_variants_keys_per_cta.txt)
  const uint64_t want = (n + FS_HIST_KEYS_PER_CTA - 1) / FS_HIST_KEYS_PER_CTA;
  const uint64_t sms = (uint64_t)device_info().sm_count;
  uint64_t g = want < sms ? want : sms;
  if (g > (uint64_t)kMaxGrid) g = kMaxGrid;
  return g ? (int)g : 1;
}

cudaError_t launch_hist16(const uint16_t* keys, uint64_t n, uint32_t* partials, unsigned long long* spill,
                          uint64_t* hist_out, uint64_t nbins_out, int accumulate, uint64_t* prefix,
                          uint64_t* slice_tot, int grid, cudaStream_t s) {
  static_assert(kHistWords % (4 * kThreads) == 0, "flush mapping");
  static_assert(kRowGroups * kSliceBins * 4 + 16 * 8 <= kHistWords * 4, "merge smem");
  // the table + one dummy word per thread + the warps' mixed-vector queues
  constexpr int smem =
      (kHistWords + kThreads) * 4 + (FS_HIST_MIXQ ? kThreads / 32 * kMixQ * 16 : 0) + (FS_HIST_HOT2W ? kThreads * 4 : 0);
  cudaError_t e = cudaFuncSetAttribute(k_hist16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  HistArgs a;
  a.keys = keys;
  a.n = n;
  // 16-byte aligned body: head keys before it, nvec full vectors, then the tail.
  const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
  a.head = ((16 - (addr & 15)) & 15) / 2;
  if (a.head > n) a.head = n;
  a.nvec = (n - a.head) / 8;
  a.partials = partials;
  a.spill = spill;
  a.hist_out = hist_out;
  a.nbins_out = nbins_out;
  a.accumulate = accumulate;
  a.prefix = prefix;
  a.slice_tot = slice_tot;
  void* args[] = {&a};
  // Cooperative launch: all CTAs co-resident (one per SM), so grid.sync() is safe.
  return cudaLaunchCooperativeKernel((const void*)k_hist16, dim3(grid), dim3(kThreads), args, smem, s);
}

}  // namespace fs
