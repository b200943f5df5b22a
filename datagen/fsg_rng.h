/*
 * fsg_rng.h — the seeded, counter-based input-generator specification.
 *
 * TEST/BENCH INFRASTRUCTURE, shared by both sides of the parity check (the
 * oracle under oracle/ and the CUDA path under paper_2605_10390_b200/).  It
 * holds none of the sorting method's arithmetic: it only turns
 * (seed, stream, global index) into a key.  Host and device include this one
 * header, so a key generated on the GPU is bit-identical to the same key
 * generated on the host (SURVEY.md §8(c).3 ledger item 18, H9).
 *
 * Generator (ledger 18): SplitMix64's output function (Steele, Lea, Flood,
 * OOPSLA 2014) applied to a Weyl sequence keyed by (seed, stream):
 *     key_s   = mix64(seed * GOLDEN + stream)
 *     draw(i) = mix64(key_s + (i + 1) * GOLDEN)
 * Everything is indexed by the GLOBAL element index i, so a shard [i0, i0+n)
 * of an N-key input is the same multiset for every way of sharding it
 * (SURVEY.md §8(e), config c4).
 */
#ifndef FSG_RNG_H
#define FSG_RNG_H
#include <stdint.h>

#if defined(__CUDACC__)
#define FSG_HD __host__ __device__ __forceinline__
#else
#define FSG_HD static inline
#endif

#define FSG_GOLDEN 0x9E3779B97F4A7C15ull

/* Streams: one per independent use of randomness. */
#define FSG_STREAM_U16 0x5531360000000001ull   /* uniform u16 keys ("U16")        */
#define FSG_STREAM_U64 0x5536340000000002ull   /* uniform u64/u32 keys ("U64")    */
#define FSG_STREAM_ZIPF 0x5A49504600000003ull  /* Zipf rank draws                 */
#define FSG_STREAM_PERM 0x5045524D00000004ull  /* Zipf value permutation          */
#define FSG_STREAM_GAUSS 0x4741555300000005ull /* Gaussian draws                  */
#define FSG_STREAM_SWAPA 0x5357504100000006ull /* sorted+swaps: first position    */
#define FSG_STREAM_SWAPB 0x5357504200000007ull /* sorted+swaps: second position   */

FSG_HD uint64_t fsg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

FSG_HD uint64_t fsg_stream_key(uint64_t seed, uint64_t stream) {
  return fsg_mix64(seed * FSG_GOLDEN + stream);
}

FSG_HD uint64_t fsg_draw_k(uint64_t stream_key, uint64_t i) {
  return fsg_mix64(stream_key + (i + 1) * FSG_GOLDEN);
}

FSG_HD uint64_t fsg_draw(uint64_t seed, uint64_t stream, uint64_t i) {
  return fsg_draw_k(fsg_stream_key(seed, stream), i);
}

/* floor(x * m / 2^64): an unbiased-enough bounded index (ledger 19/21). */
FSG_HD uint64_t fsg_mulhi64(uint64_t x, uint64_t m) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(x, m);
#else
  return (uint64_t)(((unsigned __int128)x * m) >> 64);
#endif
}

/*
 * Inverse-CDF sampling on a 65,536-entry u64 threshold table T (ledger 19/20):
 * the sample is the smallest k with draw < T[k]; T[65535] is UINT64_MAX and the
 * result is clamped to 65535.  G is a guide table: G[u] = smallest k with
 * T[k] > (u << 48), so a scan from G[draw >> 48] starts at or before the answer.
 */
FSG_HD uint32_t fsg_table_sample(const uint64_t* T, const uint32_t* G, uint64_t d) {
  uint32_t k = G[d >> 48];
  while (k < 65535u && d >= T[k]) ++k;
  return k;
}

/* Distribution ids (SURVEY.md §8(d) inputs). */
enum {
  FSG_UNIFORM = 0,     /* key = top key_bits bits of draw(U16 or U64 stream)            */
  FSG_ZIPF = 1,        /* c3a: Zipf s=1.2 over 65,536 ranks, seeded value permutation    */
  FSG_GAUSS = 2,       /* c3b: N(32768, 1024) rounded, tails folded into 0 / 65535       */
  FSG_SORTEDSWAP = 3,  /* c3c: base[i] = floor(i*65536/N) then floor(N/100) swaps       */
  FSG_CONST = 4        /* c3d: all keys 0xA5A5 (or the value passed as `param`)         */
};

#endif
