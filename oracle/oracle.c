/*
 * oracle.c — the plain CPU oracle of the hot path (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may call it; the product path never
 * does.  It is deliberately slow and literal: each function follows the plain
 * definition or the paper's algorithm in the paper's order, single-threaded,
 * with no blocking, fusion or reordering.  It shares no code, header, table or
 * helper with the CUDA path.
 *
 * Readings of the paper taken here are SURVEY.md §8(c).3 ledger items, listed
 * in DESIGN.md §Readings.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ u16 path */

void oracle_histogram_u16(const uint16_t* keys, uint64_t n, uint64_t* C) {
  /* Fractal RMW leaf level: each key increments the counter of
   * the leaf its bit path selects; at p = 16 the leaf slot is the key itself
   * (ledger 1, MSB-first; PAPER.md:197 computable pointers). */
  memset(C, 0, sizeof(uint64_t) * 65536);
  for (uint64_t i = 0; i < n; ++i) C[keys[i]] += 1;
}

void oracle_exclusive_scan_u64(const uint64_t* C, uint64_t nbins, uint64_t* P) {
  /* GetIndex(v) = number of keys strictly less than v (Alg. 3, ledger 6),
   * for every v at once; Alg. 5's running "offset <- offset + C[b]". */
  P[0] = 0;
  for (uint64_t v = 0; v < nbins; ++v) P[v + 1] = P[v] + C[v];
}

void oracle_reconstruct_counts_u16(const uint64_t* C, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                                   uint16_t* out) {
  /* Alg. 5 with t = p - l_n = 0 and l_b = 0: entries carry
   * no bits, so each bin b is reconstructed as the key b, C[b] times. */
  uint64_t offset = 0, idx = 0;
  for (uint64_t b = 0; b < nbins; ++b) {
    if (C[b] == 0) continue; /* "if C[b] = 0 continue" */
    if (offset + C[b] <= out_begin || idx >= out_end) { /* bin wholly outside the requested range */
      idx += C[b];
      offset += C[b];
      continue;
    }
    for (uint64_t s = 0; s < C[b]; ++s) {
      if (idx >= out_begin && idx < out_end) out[idx - out_begin] = (uint16_t)b;
      idx += 1;
    }
    offset += C[b];
  }
}

void oracle_sort_u16(const uint16_t* keys, uint64_t n, uint16_t* out) {
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * 65536);
  oracle_histogram_u16(keys, n, C);
  oracle_reconstruct_counts_u16(C, 65536, 0, n, out);
  free(C);
}

/* ------------------------------------------------------------ trie and queries */

int oracle_trie_levels(const uint64_t* keys, uint64_t n, int p, uint64_t* levels) {
  if (p < 1 || p > 24) return -1;
  memset(levels, 0, sizeof(uint64_t) * (((uint64_t)2 << p) - 1));
  for (uint64_t i = 0; i < n; ++i) {
    /* AddItem: node <- root; node.counter += 1; descend by the path bit,
     * MSB first (level l reads bit p-1-l, ledger 1), until the leaf level p. */
    uint64_t node = 0; /* prefix of the key consumed so far */
    for (int l = 0; l <= p; ++l) {
      levels[(((uint64_t)1 << l) - 1) + node] += 1;
      if (l < p) node = (node << 1) | ((keys[i] >> (p - 1 - l)) & 1u);
    }
  }
  return 0;
}

static uint64_t level_count(const uint64_t* levels, int l, uint64_t node) {
  return levels[(((uint64_t)1 << l) - 1) + node];
}

uint64_t oracle_get_item(const uint64_t* levels, int p, uint64_t r, uint64_t default_value) {
  /* Alg. 2 read as standard order-statistic descent (ledger 4): go left if
   * r < count(left child), else subtract count(left child) and go right; the
   * key is rebuilt from the path bits (ledger 5). */
  if (r >= level_count(levels, 0, 0)) return default_value;
  uint64_t node = 0;
  for (int l = 0; l < p; ++l) {
    const uint64_t left = node << 1;
    const uint64_t cl = level_count(levels, l + 1, left);
    if (r < cl) {
      node = left;
    } else {
      r -= cl;
      node = left | 1u;
    }
  }
  return node;
}

uint64_t oracle_get_index(const uint64_t* levels, int p, uint64_t v) {
  /* Alg. 3 (ledger 6): idx accumulates the counts of left subtrees passed on
   * the way to v, i.e. the number of keys < v. */
  uint64_t idx = 0, node = 0;
  for (int l = 0; l < p; ++l) {
    const uint64_t bit = (v >> (p - 1 - l)) & 1u;
    const uint64_t left = node << 1;
    if (bit) idx += level_count(levels, l + 1, left);
    node = left | bit;
  }
  return idx;
}

uint64_t oracle_bit_reverse(uint64_t x, int width) {
  uint64_t r = 0;
  for (int i = 0; i < width; ++i) r |= ((x >> i) & 1u) << (width - 1 - i);
  return r;
}

/* --------------------------------------------------- Alg. 5, general (p, l_b) */

static uint64_t low_mask(int bits) { return bits >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << bits) - 1); }

/* Stable argsort of seg[0..m) into I (bottom-up merge sort: stable by construction). */
static void stable_argsort_u64(const uint64_t* seg, uint64_t m, uint64_t* I, uint64_t* tmp) {
  for (uint64_t i = 0; i < m; ++i) I[i] = i;
  for (uint64_t width = 1; width < m; width *= 2) {
    for (uint64_t lo = 0; lo < m; lo += 2 * width) {
      uint64_t mid = lo + width < m ? lo + width : m;
      uint64_t hi = lo + 2 * width < m ? lo + 2 * width : m;
      uint64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = (seg[I[b]] < seg[I[a]]) ? I[b++] : I[a++];
      while (a < mid) tmp[o++] = I[a++];
      while (b < hi) tmp[o++] = I[b++];
    }
    memcpy(I, tmp, sizeof(uint64_t) * m);
  }
}

int oracle_trie_depth(uint64_t n, int p) {
  /* l_n = min(p, ceil(log2 n)); 0 for n <= 1. */
  int lg = 0;
  while (lg < 64 && ((uint64_t)1 << lg) < n) ++lg;
  return p < lg ? p : lg;
}

void oracle_decompose(uint64_t key, int p, int l_n, int l_b, uint64_t* bin, uint64_t* offset, uint64_t* trailing) {
  /* bin = top (l_n - l_b) bits, offset = next l_b bits,
   * trailing = low t = p - l_n bits (ledger 8: bins are the top bits). */
  const int t = p - l_n, bin_bits = l_n - l_b;
  *trailing = key & low_mask(t);
  *offset = (t >= 64 ? 0 : (key >> t)) & low_mask(l_b);
  *bin = bin_bits == 0 ? 0 : (key >> (l_b + t)) & low_mask(bin_bits);
}

int oracle_build_bins(const uint64_t* keys, uint64_t n, int p, int l_n, int l_b, uint64_t* C, uint64_t* E) {
  /* count keys per bin, then scatter each key's entry
   * (offset << t) | trailing to its bin's segment in arrival order. */
  const int t = p - l_n;
  if (l_n - l_b > 26 || l_b < 0 || l_b > l_n) return -1;
  const uint64_t n_bins = (uint64_t)1 << (l_n - l_b);
  uint64_t* next = (uint64_t*)malloc(sizeof(uint64_t) * n_bins);
  if (!next) return -3;
  memset(C, 0, sizeof(uint64_t) * n_bins);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t b, o, tr;
    oracle_decompose(keys[i], p, l_n, l_b, &b, &o, &tr);
    C[b] += 1;
  }
  uint64_t off = 0;
  for (uint64_t b = 0; b < n_bins; ++b) { next[b] = off; off += C[b]; }
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t b, o, tr;
    oracle_decompose(keys[i], p, l_n, l_b, &b, &o, &tr);
    E[next[b]++] = (t >= 64 ? 0 : (o << t)) | tr;
  }
  free(next);
  return 0;
}

int oracle_sort_bin(const uint64_t* seg, uint64_t m, uint64_t* I) {
  /* stable argsort of one bin's entries; I maps sorted
   * position -> arrival position within the bin. */
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
  if (!tmp) return -3;
  stable_argsort_u64(seg, m, I, tmp);
  free(tmp);
  return 0;
}

void oracle_reconstruct_all(const uint64_t* E, const uint64_t* I, const uint64_t* C, int p, int l_n, int l_b,
                            uint64_t* K) {
  /* Alg. 5 ReconstructAll, line by line.  Ledger 8: bins
   * are enumerated in ascending numeric order and the key is
   * bin || offset || trailing from MSB to LSB, so BitReverse is the identity
   * layout here. */
  const uint64_t n_bins = (uint64_t)1 << (l_n - l_b);  /* line 2 */
  const int t = p - l_n;                               /* line 2 */
  uint64_t offset = 0, idx = 0;                        /* line 3 */
  for (uint64_t b = 0; b < n_bins; ++b) {              /* line 4 */
    if (C[b] == 0) continue;                           /* line 5 */
    const uint64_t key_high = (l_n - l_b) == 0 ? 0 : (b << (l_b + t)); /* line 6 */
    for (uint64_t s = 0; s < C[b]; ++s) {              /* line 7 */
      const uint64_t entry = E[offset + I[offset + s]];           /* line 8 */
      const uint64_t trailing = entry & low_mask(t);              /* line 9 */
      const uint64_t tree_off = t >= 64 ? 0 : (entry >> t);       /* line 10 */
      const uint64_t off_val = tree_off;                          /* line 11 */
      K[idx] = key_high | (t >= 64 ? 0 : (off_val << t)) | trailing; /* line 12 */
      idx += 1;                                                   /* line 13 */
    }
    offset += C[b];                                    /* line 15 */
  }
}

int oracle_alg5_sort(const uint64_t* keys, uint64_t n, int p, int l_b, uint64_t* out, uint64_t* C_out) {
  if (p < 1 || p > 64 || l_b < 0) return -1;
  if (n == 0) return 0;
  const int l_n = oracle_trie_depth(n, p);
  if (l_b > l_n) l_b = l_n; /* 0 <= l_b <= l_n */
  if (l_n - l_b > 26) return -2; /* the oracle is for small cases */
  const uint64_t n_bins = (uint64_t)1 << (l_n - l_b);
  uint64_t* C = (uint64_t*)calloc(n_bins, sizeof(uint64_t));
  uint64_t* E = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* I = (uint64_t*)malloc(sizeof(uint64_t) * n);
  if (!C || !E || !I) return -3;
  int rc = oracle_build_bins(keys, n, p, l_n, l_b, C, E);
  uint64_t off = 0;
  for (uint64_t b = 0; b < n_bins && rc == 0; ++b) {
    rc = oracle_sort_bin(E + off, C[b], I + off);
    off += C[b];
  }
  if (rc == 0) oracle_reconstruct_all(E, I, C, p, l_n, l_b, out);
  if (rc == 0 && C_out) memcpy(C_out, C, sizeof(uint64_t) * n_bins);
  free(C);
  free(E);
  free(I);
  return rc;
}

int oracle_counter_width(int level, uint64_t capacity, int min_width) {
  /* Tapered counter width (§III.D.1, 197; ledger 11):
   * w_l = max(w_min, ceil(log2(capacity + 1)) - l). */
  int w = 0;
  while (w < 64 && (((uint64_t)1 << w) - 1) < capacity) ++w;
  w -= level;
  return w > min_width ? w : min_width;
}

/* Tapered, bit-packed export of the dense trie levels (NEXT-3 of SURVEY.md
 * §8(f)): level l gets width w_l = oracle_counter_width(l, capacity, min_width)
 * (§III.D.1), promoted by 4 bits while its largest
 * counter does not fit (SPEC.md:142 overflow policy: never wrap), capped at 64.
 * Counter i of level l occupies stream bits [off_l + i*w_l, off_l + (i+1)*w_l),
 * off_0 = 0, off_{l+1} = off_l + 2^l * w_l; stream bit b is bit (b mod 64) of
 * word b / 64 (LSB first).  Returns the number of words used, or -1 if
 * `words` is too small. */
int64_t oracle_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int* widths,
                         uint64_t* bit_offsets, uint64_t* packed, uint64_t words) {
  uint64_t off = 0;
  for (int l = 0; l <= p; ++l) {
    uint64_t mx = 0;
    for (uint64_t i = 0; i < ((uint64_t)1 << l); ++i)
      if (level_count(levels, l, i) > mx) mx = level_count(levels, l, i);
    int w = oracle_counter_width(l, capacity, min_width);
    while (w < 64 && (mx >> w) != 0) w += 4;
    if (w > 64) w = 64;
    widths[l] = w;
    bit_offsets[l] = off;
    off += ((uint64_t)1 << l) * (uint64_t)w;
  }
  bit_offsets[p + 1] = off;
  const uint64_t used = (off + 63) / 64;
  if (used > words) return -1;
  memset(packed, 0, sizeof(uint64_t) * used);
  for (int l = 0; l <= p; ++l) {
    for (uint64_t i = 0; i < ((uint64_t)1 << l); ++i) {
      const uint64_t x = level_count(levels, l, i);
      for (int b = 0; b < widths[l]; ++b) {  /* one bit at a time: obviously correct */
        const uint64_t pos = bit_offsets[l] + i * (uint64_t)widths[l] + (uint64_t)b;
        packed[pos / 64] |= ((x >> b) & 1u) << (pos % 64);
      }
    }
  }
  return (int64_t)used;
}

/* ---------------------------------------------------------- LSD pairs / keys */

int oracle_sort_pairs_u64_u32(const uint64_t* kin, const uint32_t* vin, uint64_t n, int key_bits,
                              uint64_t* kout, uint32_t* vout) {
  if (key_bits < 1 || key_bits > 64) return -1;
  if (n == 0) return 0;
  const int passes = (key_bits + 15) / 16;
  uint64_t* ka = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* kb = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint32_t* va = vin ? (uint32_t*)malloc(sizeof(uint32_t) * n) : NULL;
  uint32_t* vb = vin ? (uint32_t*)malloc(sizeof(uint32_t) * n) : NULL;
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * 65536);
  uint64_t* P = (uint64_t*)malloc(sizeof(uint64_t) * 65537);
  if (!ka || !kb || !C || !P || (vin && (!va || !vb))) return -3;
  memcpy(ka, kin, sizeof(uint64_t) * n);
  if (vin) memcpy(va, vin, sizeof(uint32_t) * n);
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 16 * pass;
    /* histogram phase */
    memset(C, 0, sizeof(uint64_t) * 65536);
    for (uint64_t i = 0; i < n; ++i) C[(ka[i] >> shift) & 0xFFFF] += 1;
    /* prefix-sum phase */
    oracle_exclusive_scan_u64(C, 65536, P);
    /* stable scatter phase: input order preserved within a digit */
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t d = (ka[i] >> shift) & 0xFFFF;
      const uint64_t dst = P[d]++;
      kb[dst] = ka[i];
      if (vin) vb[dst] = va[i];
    }
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  memcpy(kout, ka, sizeof(uint64_t) * n);
  if (vin) memcpy(vout, va, sizeof(uint32_t) * n);
  free(ka); free(kb); free(va); free(vb); free(C); free(P);
  return 0;
}

int oracle_sort_keys_u32(const uint32_t* kin, uint64_t n, int key_bits, uint32_t* kout) {
  if (key_bits < 1 || key_bits > 32) return -1;
  if (n == 0) return 0;
  uint64_t* k64 = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* o64 = (uint64_t*)malloc(sizeof(uint64_t) * n);
  if (!k64 || !o64) return -3;
  for (uint64_t i = 0; i < n; ++i) k64[i] = kin[i];
  int rc = oracle_sort_pairs_u64_u32(k64, NULL, n, key_bits, o64, NULL);
  for (uint64_t i = 0; i < n; ++i) kout[i] = (uint32_t)o64[i];
  free(k64); free(o64);
  return rc;
}

/* ------------------------------------------------------------- multi-rank */

static uint64_t range_begin(int d, int G, uint64_t N) {
  return (uint64_t)(((unsigned __int128)N * (unsigned)d) / (unsigned)G);
}

void oracle_send_counts(const uint64_t* C_all, int G, int g, uint64_t nbins, uint64_t* send) {
  uint64_t N = 0;
  for (int r = 0; r < G; ++r)
    for (uint64_t v = 0; v < nbins; ++v) N += C_all[(uint64_t)r * nbins + v];
  for (int d = 0; d < G; ++d) send[d] = 0;
  uint64_t Pv = 0; /* global exclusive prefix of bin v */
  for (uint64_t v = 0; v < nbins; ++v) {
    uint64_t below = 0; /* keys of value v on lower ranks */
    for (int r = 0; r < g; ++r) below += C_all[(uint64_t)r * nbins + v];
    const uint64_t lo = Pv + below, hi = lo + C_all[(uint64_t)g * nbins + v];
    for (int d = 0; d < G; ++d) {
      const uint64_t b0 = range_begin(d, G, N), b1 = range_begin(d + 1, G, N);
      const uint64_t a = lo > b0 ? lo : b0, b = hi < b1 ? hi : b1;
      if (b > a) send[d] += b - a;
    }
    for (int r = 0; r < G; ++r) Pv += C_all[(uint64_t)r * nbins + v];
  }
}

/* --------------------------------------------------------------- checkers */

uint64_t oracle_check_nondecreasing_u16(const uint16_t* a, uint64_t n) {
  for (uint64_t i = 1; i < n; ++i)
    if (a[i] < a[i - 1]) return i + 1;
  return 0;
}

uint64_t oracle_check_pairs_index(const uint64_t* kin, uint64_t n, const uint64_t* kout, const uint32_t* vout) {
  uint8_t* seen = (uint8_t*)calloc(n ? n : 1, 1);
  if (!seen) return ~(uint64_t)0;
  uint64_t bad = 0;
  for (uint64_t j = 0; j < n && !bad; ++j) {
    const uint64_t v = vout[j];
    if (v >= n || seen[v]) bad = j + 1;                       /* permutation */
    else if (kout[j] != kin[v]) bad = j + 1;                  /* gather consistency */
    else if (j && kout[j] < kout[j - 1]) bad = j + 1;         /* non-decreasing */
    else if (j && kout[j] == kout[j - 1] && vout[j] < vout[j - 1]) bad = j + 1; /* stability */
    if (!bad) seen[v] = 1;
  }
  free(seen);
  return bad;
}
