/*
 * fsg.h — C ABI of the seeded input generators (libfsdatagen.so).
 *
 * TEST/BENCH INFRASTRUCTURE: used by tests/, bench.py and smoke() to build the
 * synthetic inputs of SURVEY.md §8(d) (configs c1..c5 of BASELINE.json).  It is
 * neither the oracle nor the product: it holds none of the sorting method's
 * arithmetic.  Host and device generators share only fsg_rng.h, so they are
 * bit-identical by construction (and a GPU test checks it).
 *
 * All functions return 0 on success, a negative value on invalid arguments and
 * a positive CUDA error code on a CUDA failure.  `stream` is a cudaStream_t.
 * Keys are indexed by GLOBAL index: element j of `out` is key number i0 + j of
 * an n_total-key input.
 */
#ifndef FSG_H
#define FSG_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* u16 keys of distribution `dist` (FSG_* in fsg_rng.h).  key_bits in 1..16
 * applies to FSG_UNIFORM only; `param` is the constant for FSG_CONST. */
int fsg_gen_u16_host(int dist, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total,
                     int key_bits, uint32_t param, uint16_t* out);
/* Device variant; FSG_SORTEDSWAP is host-only (its swaps are sequential). */
int fsg_gen_u16_device(int dist, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total,
                       int key_bits, uint32_t param, uint16_t* out, void* stream);

/* Uniform u32/u64 keys: the top key_bits bits of draw(seed, U64, i). */
int fsg_gen_u32_host(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint32_t* out);
int fsg_gen_u64_host(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint64_t* out);
int fsg_gen_u32_device(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint32_t* out, void* stream);
int fsg_gen_u64_device(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint64_t* out, void* stream);

/* values[j] = (uint32_t)(i0 + j): config c5's "values equal the original index". */
int fsg_iota_u32_host(uint64_t i0, uint64_t n, uint32_t* out);
int fsg_iota_u32_device(uint64_t i0, uint64_t n, uint32_t* out, void* stream);

/* The inverse-CDF tables behind FSG_ZIPF / FSG_GAUSS (for tests):
 * T[65536] thresholds, G[65536] guide, perm[65536] value permutation (Zipf;
 * identity for Gauss). */
int fsg_tables(int dist, uint64_t seed, uint64_t* T, uint32_t* G, uint16_t* perm);

#ifdef __cplusplus
}
#endif
#endif
