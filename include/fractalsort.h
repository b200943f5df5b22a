/*
 * fractalsort.h — C ABI of libfractalsort.so, the B200-native (sm_100a) hot path
 * of FractalSortCPU (arXiv 2605.10390): histogram-driven radix sorting of
 * fixed-width unsigned keys with the paper's compressed histogram.
 *
 * Citations are lines of /root/reference/PAPER.md (section named) and of SPEC.md;
 * readings of ambiguous passages are the ledger items of SURVEY.md §8(c).3, listed
 * in DESIGN.md §Readings.
 *
 * Problem statement: sort n keys of precision p = key_bits
 * ascending; the output is the "Sorted array K of n reconstructed p-bit keys"
 * (Alg. 5).  For key/value pairs the sort is stable: values are the
 * paper's index array I, which "maps each sorted position to an arrival position"
 * (ledger 13).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Pointers named keys/vals/hist/prefix/out/temp are DEVICE pointers (CUDA
 *    global memory of the current device), except where a name ends in _host.
 *    The caller owns every buffer; the library allocates no memory and keeps no
 *    state except a per-device attribute cache (thread-safe) and, for
 *    fs_sort_keys_u16_host only, two copy streams and 9 events per host thread
 *    and device, created on that thread's first call and kept for the process.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    asynchronous and stream-ordered; there is no host synchronisation, so
 *    device-side faults surface at the caller's next synchronisation.  Setting
 *    the environment variable FS_SYNC_CHECK=1 makes every call synchronise and
 *    report asynchronous errors as FS_ERR_CUDA (debugging aid).
 *  - n is a 64-bit element count (up to 2^34 per device is exercised); all
 *    counts and positions are 64-bit.
 *  - n == 0 returns FS_OK without launching anything (ledger 14).
 *  - key_bits: 0 means the full key width; otherwise 1..width.  Keys must be
 *    < 2^key_bits ("key < 2^p"); violating that is a precondition
 *    error with unspecified (but memory-safe) output.  For u16 keys-only the
 *    output is the exact sort even then; key_bits only sets hist sizes.
 *  - Errors are returned, never printed or aborted on: NULL pointers with n > 0,
 *    temp_bytes smaller than the matching *_temp_bytes(), key_bits out of range,
 *    or forbidden aliasing give FS_ERR_INVALID_ARGUMENT before any CUDA call;
 *    launch failures give FS_ERR_CUDA.  fs_last_error_message() holds a
 *    thread-local detail string for the last failure on the calling thread.
 *  - Results are deterministic and bit-identical across runs, grid sizes and
 *    devices (integer arithmetic only; stability fixes the order of equal keys).
 *  - temp must be 256-byte aligned (torch / cudaMalloc allocations are).
 */
#ifndef FRACTALSORT_H
#define FRACTALSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fs_stream_t; /* == cudaStream_t */

typedef enum {
  FS_OK = 0,
  FS_ERR_INVALID_ARGUMENT = 1,
  FS_ERR_CUDA = 2,
  FS_ERR_OUT_OF_MEMORY = 3,
  FS_ERR_UNSUPPORTED = 4
} fs_status;

/* Static English name of a status code. */
const char* fs_status_string(fs_status s);
/* Thread-local detail of the last failing call on this thread ("" if none). */
const char* fs_last_error_message(void);
/* ABI version: (major << 16) | minor. */
int fs_version(void);

/* ----------------------------------------------------------------------------
 * Temp sizing.  Each returns the minimum temp_bytes for the matching call with
 * the same arguments on the current device (depends on the SM count).
 * ------------------------------------------------------------------------- */
size_t fs_sort_keys_u16_temp_bytes(uint64_t n);
size_t fs_sort_keys_u32_temp_bytes(uint64_t n, int key_bits);
size_t fs_sort_keys_u64_temp_bytes(uint64_t n, int key_bits);
size_t fs_sort_pairs_u64_u32_temp_bytes(uint64_t n, int key_bits);
size_t fs_histogram_u16_temp_bytes(uint64_t n);
size_t fs_exclusive_scan_u64_temp_bytes(uint64_t nbins);

/* ----------------------------------------------------------------------------
 * fs_sort_keys_u16 — keys-only ascending sort of n u16 keys (configs c1-c4).
 *
 * The three stages of the paper's method at p = 16, n > 2^p (the full-histogram
 * branch, §III.G; K1 of SURVEY.md §0.3):
 *   1. compressed histogram of the 65,536 leaf bins: every key increments the
 *      leaf its MSB-first bit path selects (Fractal RMW, §III.B.1;
 *      Alg. 1), in 16-bit tapered counters packed two per
 *      32-bit word (§III.D.1, 197 §III.F.1, n_L = W/w_c PAPER.md:222),
 *      per-SM local trees merged into one global histogram;
 *   2. exclusive scan P[v] = #keys < v = GetIndex(v) for all v (Alg. 3,
 *      PAPER.md:168-190);
 *   3. reconstruction = count-expansion: out[P[v] .. P[v+1]) = v (Alg. 5,
 *      PAPER.md:256-286, with t = 0 and l_b = 0).
 * n <= 2^18: the three stages run in one launch of a 16-CTA thread-block
 * cluster (per-CTA histograms merged through L2, the expansion staged in
 * shared memory); larger n: a cooperative histogram kernel and the expansion.
 * keys_in, keys_out: device arrays of n u16.  keys_out == keys_in (in place) is
 * allowed; any other overlap is FS_ERR_INVALID_ARGUMENT.  key_bits: 0 or 1..16.
 * temp: >= fs_sort_keys_u16_temp_bytes(n) device bytes (contents undefined on
 * entry and exit).
 * ------------------------------------------------------------------------- */
fs_status fs_sort_keys_u16(const uint16_t* keys_in, uint16_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * fs_sort_keys_u32 / fs_sort_keys_u64 — keys-only ascending sort of wider keys.
 * Two schemes with the same (unique) result:
 *  - trie-binned MSD (NEXT-1; n > 8,960 and key_bits >= 32): one read builds the
 *    leaf level of a 16-level compressed trie over the top 16 key bits; its
 *    level-8 and level-16 counters bound two stable 8-bit MSD scatters; every
 *    16-bit bin is then sorted by its remaining bits in shared memory (Alg. 5's
 *    bins and per-bin sort).  A bin above 8,704 keys
 *    recurses on the next 8-bit digits (stable MSD scatters of its own) until
 *    every piece fits.  If the keys share a prefix (the bits where some keys
 *    differ end at hb < key_bits - 1) and hb + 1 >= 32, the 16 bins' window is
 *    moved to [hb - 15, hb] (the trie histogram is rebuilt there).  With fewer
 *    than 32 varying bits the LSD scheme below is taken — all decided on the
 *    device, no host synchronisation;
 *  - otherwise stable LSD radix ("histogram, prefix sum and stable scatter
 *    phases", §II) with 8-bit digits and one compressed histogram
 *    per digit, all digit histograms in one read pass (config c5's "multi-digit
 *    precision scaling with compressed histograms per digit", ledger 25); a
 *    digit whose histogram has one non-empty bin is skipped.  n <= 8,960 (or
 *    n <= 16,384 with key_bits < 32): the same LSD inside one CTA's shared
 *    memory (one launch).
 * keys_in and keys_out must not overlap.  key_bits: 0 or 1..32 (u32), 0 or
 * 1..64 (u64).
 * ------------------------------------------------------------------------- */
fs_status fs_sort_keys_u32(const uint32_t* keys_in, uint32_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream);
fs_status fs_sort_keys_u64(const uint64_t* keys_in, uint64_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * fs_sort_pairs_u64_u32 — STABLE ascending sort of (u64 key, u32 value) pairs
 * by key (config c5).  Equal keys keep their input order, so with
 * vals_in[i] = i the output values are Alg. 5's index array I.
 * Same schemes as fs_sort_keys_u64; keys and values move together.
 * No input buffer may overlap an output buffer.
 * ------------------------------------------------------------------------- */
fs_status fs_sort_pairs_u64_u32(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                                uint32_t* vals_out, uint64_t n, int key_bits, void* temp, size_t temp_bytes,
                                fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * Phase API (batch streaming with histogram reuse, and the multi-GPU driver).
 *
 * fs_histogram_u16: hist[v] (+)= #{i : keys[i] == v} for v < 2^key_bits (device
 * u64 array of 2^key_bits entries).  accumulate = 1 adds to the existing hist —
 * the "cached histogram from a terminating batch is reused by the next batch"
 * of Batch Counter Update (§III.D); accumulate = 0 overwrites.
 * hist may be reinterpreted by the caller as int64 (counts < 2^63).
 * ------------------------------------------------------------------------- */
fs_status fs_histogram_u16(const uint16_t* keys, uint64_t n, int key_bits, uint64_t* hist, int accumulate,
                           void* temp, size_t temp_bytes, fs_stream_t stream);

/* fs_histogram_prefix_u16 / fs_expand_prefix_u16: the sort's own two-level
 * prefix, exported for the multi-GPU path (SURVEY.md §8(e) Mode B).  prefix2
 * holds 65,536 + 128 u64: prefix2[v] = #keys < v inside v's 512-bin slice
 * (slice-local GetIndex, Alg. 3) and prefix2[65536 + s] = the total of slice s.
 * Both parts are linear in the counts, so the element-wise sum over ranks
 * (one all-reduce) is the same form for the union of the shards; expansion of
 * global positions [out_begin, out_end) then needs no scan kernel (the slice
 * bases are folded into the expansion).  temp as for
 * fs_histogram_u16; keys 2-byte aligned; the buffers must not overlap. */
fs_status fs_histogram_prefix_u16(const uint16_t* keys, uint64_t n, uint64_t* prefix2, void* temp, size_t temp_bytes,
                                  fs_stream_t stream);
fs_status fs_expand_prefix_u16(const uint64_t* prefix2, uint64_t out_begin, uint64_t out_end, uint16_t* out,
                               fs_stream_t stream);

/* fs_exclusive_scan_u64: prefix[v] = sum_{u<v} hist[u] for v = 0..nbins, so
 * prefix[nbins] is the total (Alg. 3 GetIndex for every v).
 * hist: nbins u64; prefix: nbins + 1 u64; they must not overlap.  Single-pass
 * decoupled-lookback scan.  nbins >= 1; runs even for a zero total. */
fs_status fs_exclusive_scan_u64(const uint64_t* hist, uint64_t* prefix, uint64_t nbins, void* temp,
                                size_t temp_bytes, fs_stream_t stream);

/* fs_expand_u16: count-expansion of a prefix array (Alg. 5 with t = 0, l_b = 0,
 * PAPER.md:259-284): writes the keys at global sorted positions
 * [out_begin, out_end) to out[0 .. out_end - out_begin), where the key at
 * position j is the v with prefix[v] <= j < prefix[v+1].  prefix: nbins + 1
 * non-decreasing u64 (nbins <= 65536) with out_end <= prefix[nbins].
 * This is how a rank of the multi-GPU path writes its own output range
 * (SURVEY.md §8(e) Mode B).  No temp needed. */
fs_status fs_expand_u16(const uint64_t* prefix, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                        uint16_t* out, fs_stream_t stream);

/* fs_send_counts: multi-GPU payload exchange plan (SURVEY.md §8(e) Mode A,
 * ledger 13, 23).  hist_all: G x nbins u64 (row r = rank r's histogram, as
 * gathered).  Rank d owns global sorted positions [floor(d*N/G),
 * floor((d+1)*N/G)), N = total; rank g's keys of value v occupy positions
 * [P[v] + S_<g[v], P[v] + S_<=g[v]) (lower rank first).  Writes
 * send[d] = number of rank g's keys that land in rank d's range (G u64, device).
 * G in 1..1024, 0 <= g < G, nbins <= 65536. */
fs_status fs_send_counts(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint64_t* send,
                         fs_stream_t stream);

/* fs_bound_u64: out[i] = #{j : sorted[j] < queries[i]} (upper = 0, the lower
 * bound) or #{j : sorted[j] <= queries[i]} (upper = 1) for an ascending u64
 * array of n keys on the device; q queries, one thread each.  The rank counts
 * behind the exact, sampling-free splitters of the distributed pair sort
 * (SURVEY.md §8(e) Mode A for pairs; GetIndex, Alg. 3, on a
 * sorted shard).  out must not overlap the inputs. */
fs_status fs_bound_u64(const uint64_t* sorted, uint64_t n, const uint64_t* queries, uint64_t q, int upper,
                       uint64_t* out, fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * Distributed pair sort (SURVEY.md §8(e) pairs; NEXT-2, exchange.cu).
 *
 * Exact splitters by compressed histograms (PAPER.md:95 Fractal RMW, 168-190
 * GetIndex; ledger 13, 23): the key K_d at global position s_d = floor(dN/G) is
 * fixed digit by digit, 16 bits per level, from the all-reduced histograms below.
 *
 * fs_histogram16_u64: hist[v] = #{i : ((keys[i] >> shift) & (2^width - 1)) == v}
 * for v < 2^width (u64 counts, overwritten), 1 <= width <= 16, shift + width
 * <= 64 -- the level-1 histogram over every key of the shard.  temp:
 * fs_histogram16_u64_temp_bytes(n) bytes, 256-byte aligned.
 *
 * fs_select_bins_u64: appends to out (capacity cap) every key whose digit is one
 * of bins[0..nb) (device u32, nb <= 64), in no particular order; *count
 * (device u64) receives the number of such keys (also when above cap: then only
 * cap are written).  The candidates of the later levels.
 *
 * fs_digit_counts_sorted_u64: for an ascending array sorted[0..m) and np
 * prefixes (device u64), hist[j * 2^width + v] = #{i : (sorted[i] >> shift) ==
 * (prefixes[j] >> shift) | v}: the histogram of the next digit among the keys
 * that share prefix j's bits above it (two binary searches per (j, v)).
 *
 * The fused exchange (no local sort before it, no staging copy, no all-to-all):
 * every pair gets a class, 2d for K_{d-1} < key < K_d and 2d + 1 for key == K_d
 * (the lowest such d; splitters ascending, G - 1 of them on the device); in
 * class order, stable within a class, owner d's share is one range
 * [cuts[d], cuts[d+1]).  fs_pair_classes_u64 counts the classes per 2,048-pair
 * tile, scans them into temp and writes class_tot[2G - 1] (device u64);
 * fs_pair_scatter_u64_u32 (same temp, same splitters, called after) writes
 * pair i with class-order index Q, cuts[d] <= Q < cuts[d+1], to
 * dest_keys[d][bases[d] + Q - cuts[d]] and dest_vals[...] -- dest_*: HOST arrays
 * of G device pointers (normally peer-mapped via CUDA IPC); cuts (G + 1, from 0
 * to n, ascending) and bases (G) are HOST arrays.  1 <= G <= 16.  temp:
 * fs_pair_exchange_temp_bytes(n, G) bytes, 256-byte aligned.
 * ------------------------------------------------------------------------- */
size_t fs_histogram16_u64_temp_bytes(uint64_t n);
fs_status fs_histogram16_u64(const uint64_t* keys, uint64_t n, int shift, int width, uint64_t* hist, void* temp,
                             size_t temp_bytes, fs_stream_t stream);
fs_status fs_select_bins_u64(const uint64_t* keys, uint64_t n, int shift, int width, const uint32_t* bins, int nb,
                             uint64_t* out, uint64_t cap, uint64_t* count, fs_stream_t stream);
fs_status fs_digit_counts_sorted_u64(const uint64_t* sorted, uint64_t m, const uint64_t* prefixes, int np, int shift,
                                     int width, uint64_t* hist, fs_stream_t stream);
size_t fs_pair_exchange_temp_bytes(uint64_t n, int G);
fs_status fs_pair_classes_u64(const uint64_t* keys, uint64_t n, const uint64_t* splitters, int G, uint64_t* class_tot,
                              void* temp, size_t temp_bytes, fs_stream_t stream);
fs_status fs_pair_scatter_u64_u32(const uint64_t* keys, const uint32_t* vals, uint64_t n, const uint64_t* splitters,
                                  int G, const uint64_t* cuts_host, const uint64_t* bases_host,
                                  uint64_t* const* dest_keys_host, uint32_t* const* dest_vals_host, void* temp,
                                  size_t temp_bytes, fs_stream_t stream);

/* fs_expand_to_peers_u16: the fused exchange of the multi-GPU keys-only sort
 * (SURVEY.md §8(f) NEXT-2): rank g writes each of its own keys straight to its
 * final global sorted position, in the output buffer of the rank that owns it.
 * hist_all: G x nbins u64 on the device (row r = rank r's histogram, as
 * gathered).  With N = total and P = exclusive scan of sum_r C_r, rank g's keys
 * of value v go to global positions [P[v] + S_<g[v], P[v] + S_<=g[v]) (lower
 * rank first), and rank d owns positions [floor(dN/G),
 * floor((d+1)N/G)) (ledger 23): dest[d] (a HOST array of G device pointers,
 * each dest[d] a device — normally peer-mapped via CUDA IPC — buffer of at
 * least floor((d+1)N/G) - floor(dN/G) u16) receives them at offset
 * position - floor(dN/G).  After every rank's call has completed (synchronise,
 * then a barrier across ranks), each rank's buffer holds its slice of the sorted
 * output: Alg. 5 count-expansion done by the producers.
 * temp: fs_expand_to_peers_u16_temp_bytes(nbins, G) device bytes.  The call
 * returns when the work is enqueued (dest is copied to the device in order). */
size_t fs_expand_to_peers_u16_temp_bytes(uint64_t nbins, int G);
fs_status fs_expand_to_peers_u16(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint16_t* const* dest,
                                 void* temp, size_t temp_bytes, fs_stream_t stream);

/* fs_allreduce_multicast_u64: the cross-GPU histogram merge through NVSwitch
 * multicast (NVLS; SURVEY.md §8(f) NEXT-2, row a3 across GPUs): the Global
 * Histogram Update of PAPER.md:91-92 (§III.B) over G ranks.
 * dst[i] = sum over ranks r of src_r[i] for i < count, where src_mc is the
 * MULTICAST address (cuMulticastCreate + cuMulticastBindMem, every rank's own
 * physical memory bound at the same offset) of the ranks' u64 arrays: each
 * element is one multimem.ld_reduce.add, summed by the switch.  dst: count u64
 * of ordinary device memory of the calling rank.  The call contains the
 * barrier the reduction needs: it adds 1 to the u32 flag in every rank's copy
 * (flag_mc: its multicast address, multimem.red.release) and waits until this
 * rank's copy (flag_local: the same word through the rank's unicast mapping)
 * reaches `target` (wrap-safe compare; callers pass G x the number of calls made
 * so far on this flag, this one included), so no rank reads before every rank's
 * src_r is complete.  A caller that rewrites src before every rank has read it
 * must alternate two src regions by call parity.  All pointers device, 8-byte
 * (flags 4-byte) aligned; src_mc and dst must not overlap.  Every rank of the
 * multicast group must make the matching call; a rank whose peers have not all
 * arrived within timeout_ns (0: wait forever) stops waiting, leaves dst
 * unwritten and sets the device word *timed_out to 1 (callers zero it first and
 * read it after synchronising).  count = 0 still arrives and waits (a pure
 * barrier).  Errors: FS_ERR_INVALID_ARGUMENT for NULL / misaligned /
 * overlapping arguments; FS_ERR_CUDA if the launch fails (e.g. src_mc not a
 * multicast mapping surfaces as an asynchronous fault at the caller's next
 * sync). */
fs_status fs_allreduce_multicast_u64(const uint64_t* src_mc, uint64_t* dst, uint64_t count, uint32_t* flag_mc,
                                     const uint32_t* flag_local, uint32_t target, uint64_t timeout_ns,
                                     uint32_t* timed_out, fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * Host-buffer entry point (end-to-end use, and the out-of-core path of Batch
 * Size Selection / Batch Counter Update): sorts n u16 keys
 * that live in HOST memory into a host output array.  The input streams to the
 * device in batches of `batch` keys, each histogrammed into one reused
 * histogram as it lands (copy of batch i+1 overlaps the histogram of batch i);
 * then the output is expanded batch by batch and streamed back (expansion of
 * batch j+1 overlaps the copy-out of batch j).  keys_in_host / keys_out_host
 * should be page-locked for full PCIe/C2C overlap (pageable memory works but
 * serialises copies).  work: device workspace of
 * fs_sort_keys_u16_host_work_bytes(n, batch) bytes.  batch = 0 picks a default.
 * The call returns when the work is enqueued; synchronise `stream` before
 * reading keys_out_host.  The copies run on two copy streams of the library's
 * (host-to-device and device-to-host, one pair per host thread and device,
 * created on first use and reused), so calls issued on DIFFERENT streams, each
 * with its own work buffer and output, overlap one call's copy-out with the
 * next call's copy-in (both PCIe directions busy); calls on one stream run in
 * order.  If the call fails after enqueuing work, `stream` is still made to
 * wait for every copy already queued, so later work on `stream` never races
 * them.
 * ------------------------------------------------------------------------- */
size_t fs_sort_keys_u16_host_work_bytes(uint64_t n, uint64_t batch);
fs_status fs_sort_keys_u16_host(const uint16_t* keys_in_host, uint16_t* keys_out_host, uint64_t n,
                                uint64_t batch, void* work, size_t work_bytes, fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * Order-statistic service on the compressed histogram:
 * quantiles, ranks and splitters without sorting.
 *
 * fs_trie_levels: the dense trie of a leaf histogram.  leaf_hist: 2^p u64
 * counts (e.g. fs_histogram_u16's output, p = key_bits); levels: receives
 * fs_trie_levels_count(p) = 2^(p+1) - 1 u64, level l (0 = root) at offset
 * 2^l - 1, node i of level l = #keys whose top l bits (MSB-first, ledger 1)
 * equal i = the sum of its two children (Alg. 1 PAPER.md:113-139 with the
 * SIBLING SUM of SPEC.md:127; dense computable-pointer layout, Alg. 4
 * PAPER.md:196-215).  p in 1..24; the buffers must not overlap.
 * ------------------------------------------------------------------------- */
size_t fs_trie_levels_count(int p);
fs_status fs_trie_levels(const uint64_t* leaf_hist, int p, uint64_t* levels, fs_stream_t stream);

/* fs_trie_pack: tapered, bit-packed export of the levels (counter-width
 * compression, §III.D.1): level l gets
 * w_l = max(min_width, ceil(log2(capacity + 1)) - l), promoted by +4 bits while
 * its largest counter does not fit, capped at 64 (never wrap, SPEC.md:142;
 * ledger 12).  Counter i of level l occupies stream bits
 * [off_l + i w_l, off_l + (i+1) w_l), off_0 = 0, off_{l+1} = off_l + 2^l w_l;
 * stream bit b is bit (b mod 64) of packed[b / 64].  Device outputs: widths
 * (p+1 int32), bit_offsets (p+2 u64), packed (packed_words u64, zeroed and
 * written).  capacity should be >= the total count (the root); then
 * fs_trie_pack_words(p, capacity) words always suffice.  If the stream does not
 * fit in packed_words, widths[0] is set to -1 and packed is left zeroed.
 * temp: fs_trie_pack_temp_bytes(p) device bytes.  min_width in 1..64. */
size_t fs_trie_pack_words(int p, uint64_t capacity);
size_t fs_trie_pack_temp_bytes(int p);
fs_status fs_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int32_t* widths,
                       uint64_t* bit_offsets, uint64_t* packed, uint64_t packed_words, void* temp,
                       size_t temp_bytes, fs_stream_t stream);

/* Batched queries on a packed trie (as written by fs_trie_pack), q queries, one
 * thread each, every array on the device:
 *   fs_get_item:  items[k] = the key at ascending sorted rank ranks[k] (0-based),
 *                 or default_value if ranks[k] >= total — Alg. 2 GetItem
 *                  as order-statistic descent on the LEFT
 *                 child's count (ledger 4), the key rebuilt from the path (ledger 5);
 *   fs_get_index: indices[k] = #keys < values[k] — Alg. 3 GetIndex
 *                 (ledger 6); values[k] must be < 2^p (only
 *                 the low p bits are walked otherwise). */
fs_status fs_get_item(const int32_t* widths, const uint64_t* bit_offsets, const uint64_t* packed, int p,
                      const uint64_t* ranks, uint64_t q, uint64_t default_value, uint64_t* items,
                      fs_stream_t stream);
fs_status fs_get_index(const int32_t* widths, const uint64_t* bit_offsets, const uint64_t* packed, int p,
                       const uint64_t* values, uint64_t q, uint64_t* indices, fs_stream_t stream);

/* fs_hist_merge_u64: out[i] = a[i] + b[i] for i < count — the merge of two
 * histograms (or two dense tries) "aggregated into a single ... tree"
 * (§III.A.1).  out may alias a or b. */
fs_status fs_hist_merge_u64(const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t count,
                            fs_stream_t stream);

/* ----------------------------------------------------------------------------
 * Phase instrumentation (measurement).  events: array of
 * `count` cudaEvent_t handles (created by the caller), or NULL to disable.
 * While set, the sort calls made on THIS thread record events[i] on their
 * stream at phase boundaries, i < count:
 *   fs_sort_keys_u16:  [0] start, [1] after zeroing the temp counters, [2] after
 *                      the histogram+merge+scan kernel, [3] after the expansion
 *                      kernel;
 *   wide sorts, MSD planned (n >= 2^15, key_bits >= 32): [0] start, [1] after
 *                      the trie histogram + scan + plan, [2] level-1 scatter,
 *                      [3] level-2 scatter, [4] k_heavy: level 2 of uneven
 *                      first-level buckets and the recursion into the bins
 *                      above the local-sort capacity (returns at once if there
 *                      is neither), [5] per-bin sorts, [6] after the LSD digit
 *                      histograms (they return at once when MSD ran), [7 + p]
 *                      after LSD pass p, last after the identity copy;
 *   wide sorts, LSD only: [0] start, [1] after the digit histograms + plan,
 *                      [2 + p] after scatter pass p (passes ceil(key_bits/8)),
 *                      last after the identity copy check.
 * The library does not own or destroy the events.  Returns FS_OK.
 * ------------------------------------------------------------------------- */
fs_status fs_set_phase_events(void* const* events, int count);

#ifdef __cplusplus
}
#endif
#endif /* FRACTALSORT_H */
