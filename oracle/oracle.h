/*
 * oracle.h — the plain, slow, obviously-correct CPU oracle (liboracle.so).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call it.  It
 * shares no code with the CUDA path (paper_2605_10390_b200/), and neither side
 * includes or links the other.  Citations: PAPER.md / SPEC.md line numbers
 * under /root/reference (section named beside each).
 *
 * Every result here is an exact integer result; there is no floating point.
 * Parity status of each function is recorded in DESIGN.md §Oracle; all
 * functions are pinned by tests/test_oracle_pins.py except where noted.
 */
#ifndef FS_ORACLE_H
#define FS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* C[v] = #{i : keys[i] == v}, v < 2^16.  The leaf level of the Fractal RMW
 * (§III.B.1) at p = 16, where n > 2^p makes the trie the full
 * histogram (§III.G). */
void oracle_histogram_u16(const uint16_t* keys, uint64_t n, uint64_t* C /*65536*/);

/* P[v] = sum_{u<v} C[u] for v = 0..nbins (P[nbins] = total): GetIndex(v) =
 * #keys < v for every v (Alg. 3, ledger 6). */
void oracle_exclusive_scan_u64(const uint64_t* C, uint64_t nbins, uint64_t* P /*nbins+1*/);

/* Alg. 5 ReconstructAll with t = 0 and l_b = 0 (bins =
 * leaves, entries empty): emit bin value b exactly C[b] times in ascending b.
 * Only sorted positions [out_begin, out_end) are written, to out[0..). */
void oracle_reconstruct_counts_u16(const uint64_t* C, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                                   uint16_t* out);

/* Keys-only ascending sort of u16 keys = histogram then ReconstructAll. */
void oracle_sort_u16(const uint16_t* keys, uint64_t n, uint16_t* out);

/* The same sort on nthreads POSIX threads (oracle_mt.c), for timing only:
 * private per-thread histograms, their sum, then every thread reconstructs its
 * own range of output positions (the paper's local -> global scheme,
 * PAPER.md:86-92).  Returns 0; 1 if memory is short, 2 if a thread failed. */
int oracle_sort_u16_mt(const uint16_t* keys, uint64_t n, uint16_t* out, int nthreads);

/* Alg. 1 AddItem with ledger fixes 1-3: every node on the
 * MSB-first root-to-leaf path of each key is incremented once.  levels holds
 * p+1 dense levels (computable pointers): level l has 2^l
 * counters at offset 2^l - 1.  p <= 24. */
int oracle_trie_levels(const uint64_t* keys, uint64_t n, int p, uint64_t* levels /*2^(p+1)-1*/);

/* Alg. 2 GetItem, ledger 4-5: key at sorted rank r, or
 * default_value if r >= n.  Reads the levels built above. */
uint64_t oracle_get_item(const uint64_t* levels, int p, uint64_t r, uint64_t default_value);

/* Alg. 3 GetIndex, ledger 6: #keys < v by a root-to-leaf
 * walk that adds the left-child count whenever the path goes right. */
uint64_t oracle_get_index(const uint64_t* levels, int p, uint64_t v);

/* SPEC.md:189-197 BitReverse of the low `width` bits (Alg. 5 utility). */
uint64_t oracle_bit_reverse(uint64_t x, int width);

/* The paper's general pipeline, step by step (PAPER.md:256-286, SPEC.md:164-227,
 * ledger 8-10).  l_n = oracle_trie_depth(n, p) = min(p, ceil(log2 n)),
 * t = p - l_n, l_b clamped to l_n; bins = top (l_n - l_b) bits.
 *   oracle_decompose     SPEC.md:179-187  key -> (bin, offset, trailing)
 *   oracle_build_bins    SPEC.md:199-207  C[n_bins] counts, E[n] entries (offset<<t)|trailing by bin, arrival order
 *   oracle_sort_bin      SPEC.md:209-217  stable argsort of one bin's entries -> I
 *   oracle_reconstruct_all  Alg. 5 lines 2-15 -> K (ascending, ledger 8)
 *   oracle_alg5_sort     the composition; writes the ascending sort of keys
 *                        (p <= 64 bits) and C (size 2^(l_n-l_b)) if C_out != NULL. */
int oracle_trie_depth(uint64_t n, int p);
void oracle_decompose(uint64_t key, int p, int l_n, int l_b, uint64_t* bin, uint64_t* offset, uint64_t* trailing);
int oracle_build_bins(const uint64_t* keys, uint64_t n, int p, int l_n, int l_b, uint64_t* C, uint64_t* E);
int oracle_sort_bin(const uint64_t* seg, uint64_t m, uint64_t* I);
void oracle_reconstruct_all(const uint64_t* E, const uint64_t* I, const uint64_t* C, int p, int l_n, int l_b,
                            uint64_t* K);
int oracle_alg5_sort(const uint64_t* keys, uint64_t n, int p, int l_b, uint64_t* out, uint64_t* C_out);

/* Tapered counter width w_l = max(min_width, ceil(log2(capacity+1)) - level)
 * (§III.D.1, 197 §III.F.1; ledger 11). */
int oracle_counter_width(int level, uint64_t capacity, int min_width);

/* Tapered, bit-packed export of the dense levels (NEXT-3):
 * w_l = counter_width(l, capacity, min_width) promoted by +4 until the level's
 * largest counter fits (<= 64); counter i of level l at stream bits
 * [off_l + i w_l, off_l + (i+1) w_l), LSB-first in u64 words.  widths: p+1,
 * bit_offsets: p+2.  Returns words used, -1 if `words` is too small. */
int64_t oracle_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int* widths,
                         uint64_t* bit_offsets, uint64_t* packed, uint64_t words);

/* Stable LSD radix sort ("histogram, prefix sum and stable scatter phases",
 * PAPER.md:52) with 16-bit digits over the low key_bits bits.
 * vals may be NULL (keys-only).  Each pass: count, exclusive scan, stable
 * scatter in input order. */
int oracle_sort_pairs_u64_u32(const uint64_t* kin, const uint32_t* vin, uint64_t n, int key_bits,
                              uint64_t* kout, uint32_t* vout);
int oracle_sort_keys_u32(const uint32_t* kin, uint64_t n, int key_bits, uint32_t* kout);

/* Exact multi-rank output partition (ledger 13, 23): rank d
 * owns global sorted positions [floor(d*N/G), floor((d+1)*N/G)).  Keys of rank
 * g with value v occupy global positions [P[v] + S_{<g}[v], P[v] + S_{<=g}[v])
 * (lower rank first).  send[d] = how many of rank g's keys land in
 * rank d's range.  C_all is G x nbins (row-major). */
void oracle_send_counts(const uint64_t* C_all, int G, int g, uint64_t nbins, uint64_t* send /*G*/);

/* Invariant checkers.  Return 0 when the property
 * holds, else 1 + the first offending index (saturated). */
uint64_t oracle_check_nondecreasing_u16(const uint16_t* a, uint64_t n);
/* Pairs produced from vals_in[i] = i: keys non-decreasing, vals_out a
 * permutation of 0..n-1, keys_out[j] == keys_in[vals_out[j]], and equal keys
 * keep ascending vals (stability).  Returns 0 when all hold. */
uint64_t oracle_check_pairs_index(const uint64_t* kin, uint64_t n, const uint64_t* kout, const uint32_t* vout);

#ifdef __cplusplus
}
#endif
#endif
