/*
 * datagen.cu — host and device implementations of the seeded input generators
 * declared in fsg.h.  TEST/BENCH INFRASTRUCTURE (see fsg.h); shares only
 * fsg_rng.h between the two sides.
 *
 * Distribution recipes (SURVEY.md §8(c).3 ledger items 18-22, §8(d)):
 *   uniform   key = draw(seed, U16, i) >> (64 - key_bits)
 *   zipf      rank k = inverse-CDF of P(r) ∝ r^-1.2, r = 1..65536 (long double
 *             thresholds); key = perm[k], perm a Fisher-Yates shuffle driven by
 *             the PERM stream with mulhi64-bounded indices
 *   gauss     k = round(N(32768, 1024)), tails folded into 0 and 65535: exact
 *             discretised CDF via erfcl, sampled by inverse-CDF
 *   sorted+swaps  base[i] = floor(i*65536/N); then floor(N/100) sequential swaps
 *             of (mulhi(draw(SWAPA,s),N), mulhi(draw(SWAPB,s),N)), s = 0,1,...
 *   const     every key = param (0xA5A5 for config c3d, ledger 22)
 */
#include <cuda_runtime.h>
#include <math.h>
#include <mutex>
#include <stdlib.h>
#include <string.h>

#include "fsg.h"
#include "fsg_rng.h"

namespace {

constexpr int kNumValues = 65536;

void build_threshold_table(const long double* cdf, uint64_t* T) {
  const long double two64 = 18446744073709551616.0L;
  for (int k = 0; k < kNumValues; ++k) {
    long double x = cdf[k] * two64;
    if (k == kNumValues - 1 || x >= two64)
      T[k] = UINT64_MAX;
    else if (x <= 0)
      T[k] = 0;
    else
      T[k] = (uint64_t)x;
  }
  T[kNumValues - 1] = UINT64_MAX;
}

void build_guide(const uint64_t* T, uint32_t* G) {
  uint32_t k = 0;
  for (uint32_t u = 0; u < (uint32_t)kNumValues; ++u) {
    const uint64_t lo = (uint64_t)u << 48;
    while (k < (uint32_t)kNumValues - 1 && T[k] <= lo) ++k;
    G[u] = k;
  }
}

int host_tables(int dist, uint64_t seed, uint64_t* T, uint32_t* G, uint16_t* perm) {
  long double* cdf = (long double*)malloc(sizeof(long double) * kNumValues);
  if (!cdf) return -2;
  if (dist == FSG_ZIPF) {
    long double H = 0;
    for (int r = kNumValues; r >= 1; --r) H += powl((long double)r, -1.2L);
    long double cum = 0;
    for (int k = 0; k < kNumValues; ++k) {
      cum += powl((long double)(k + 1), -1.2L);
      cdf[k] = cum / H;
    }
    for (int v = 0; v < kNumValues; ++v) perm[v] = (uint16_t)v;
    const uint64_t ks = fsg_stream_key(seed, FSG_STREAM_PERM);
    for (uint32_t i = kNumValues - 1, s = 0; i >= 1; --i, ++s) {
      const uint32_t j = (uint32_t)fsg_mulhi64(fsg_draw_k(ks, s), (uint64_t)i + 1);
      const uint16_t t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
  } else if (dist == FSG_GAUSS) {
    const long double mu = 32768.0L, sigma = 1024.0L;
    for (int k = 0; k < kNumValues; ++k) {
      const long double x = ((long double)k + 0.5L - mu) / sigma;
      cdf[k] = 0.5L * erfcl(-x / sqrtl(2.0L));
    }
    for (int v = 0; v < kNumValues; ++v) perm[v] = (uint16_t)v;
  } else {
    free(cdf);
    return -1;
  }
  build_threshold_table(cdf, T);
  build_guide(T, G);
  free(cdf);
  return 0;
}

inline uint16_t u16_key(int dist, uint64_t ks, uint64_t i, int key_bits, uint32_t param,
                        const uint64_t* T, const uint32_t* G, const uint16_t* perm) {
  switch (dist) {
    case FSG_UNIFORM: return (uint16_t)(fsg_draw_k(ks, i) >> (64 - key_bits));
    case FSG_ZIPF: return perm[fsg_table_sample(T, G, fsg_draw_k(ks, i))];
    case FSG_GAUSS: return (uint16_t)fsg_table_sample(T, G, fsg_draw_k(ks, i));
    default: return (uint16_t)param;
  }
}

uint64_t stream_for(int dist) {
  return dist == FSG_ZIPF ? FSG_STREAM_ZIPF : dist == FSG_GAUSS ? FSG_STREAM_GAUSS : FSG_STREAM_U16;
}

// ---------------------------------------------------------------- device side
struct DevTables {
  uint64_t seed = 0;
  int dist = -1;
  uint64_t* T = nullptr;
  uint32_t* G = nullptr;
  uint16_t* perm = nullptr;
};
std::mutex g_mu;
DevTables g_dev[64];

__global__ void k_gen_u16(int dist, uint64_t ks, uint64_t i0, uint64_t n, int key_bits, uint32_t param,
                          const uint64_t* __restrict__ T, const uint32_t* __restrict__ G,
                          const uint16_t* __restrict__ perm, uint16_t* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + j;
    uint16_t key;
    if (dist == FSG_UNIFORM)
      key = (uint16_t)(fsg_draw_k(ks, i) >> (64 - key_bits));
    else if (dist == FSG_ZIPF)
      key = perm[fsg_table_sample(T, G, fsg_draw_k(ks, i))];
    else if (dist == FSG_GAUSS)
      key = (uint16_t)fsg_table_sample(T, G, fsg_draw_k(ks, i));
    else
      key = (uint16_t)param;
    out[j] = key;
  }
}

template <typename K>
__global__ void k_gen_wide(uint64_t ks, uint64_t i0, uint64_t n, int key_bits, K* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = (K)(fsg_draw_k(ks, i0 + j) >> (64 - key_bits));
}

__global__ void k_iota(uint64_t i0, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = (uint32_t)(i0 + j);
}

int grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g ? (int)g : 1;
}

int cuda_rc(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

}  // namespace

extern "C" {

int fsg_tables(int dist, uint64_t seed, uint64_t* T, uint32_t* G, uint16_t* perm) {
  if (!T || !G || !perm) return -1;
  return host_tables(dist, seed, T, G, perm);
}

int fsg_gen_u16_host(int dist, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total, int key_bits,
                     uint32_t param, uint16_t* out) {
  if (n && !out) return -1;
  if (key_bits < 1 || key_bits > 16) return -1;
  if (dist == FSG_SORTEDSWAP) {
    // The swaps are a sequential process over the whole N-key array, so only a
    // full array (i0 == 0, n == n_total) is defined.
    if (i0 != 0 || n != n_total) return -1;
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint16_t)((i * 65536ull) / n);
    const uint64_t ka = fsg_stream_key(seed, FSG_STREAM_SWAPA);
    const uint64_t kb = fsg_stream_key(seed, FSG_STREAM_SWAPB);
    const uint64_t swaps = n / 100;
    for (uint64_t s = 0; s < swaps; ++s) {
      const uint64_t a = fsg_mulhi64(fsg_draw_k(ka, s), n);
      const uint64_t b = fsg_mulhi64(fsg_draw_k(kb, s), n);
      const uint16_t t = out[a];
      out[a] = out[b];
      out[b] = t;
    }
    return 0;
  }
  if (dist < 0 || dist > FSG_CONST) return -1;
  uint64_t* T = nullptr;
  uint32_t* G = nullptr;
  uint16_t* perm = nullptr;
  if (dist == FSG_ZIPF || dist == FSG_GAUSS) {
    T = (uint64_t*)malloc(8 * kNumValues);
    G = (uint32_t*)malloc(4 * kNumValues);
    perm = (uint16_t*)malloc(2 * kNumValues);
    if (!T || !G || !perm) return -2;
    int rc = host_tables(dist, seed, T, G, perm);
    if (rc) return rc;
  }
  const uint64_t ks = fsg_stream_key(seed, stream_for(dist));
  for (uint64_t j = 0; j < n; ++j) out[j] = u16_key(dist, ks, i0 + j, key_bits, param, T, G, perm);
  free(T);
  free(G);
  free(perm);
  return 0;
}

int fsg_gen_u16_device(int dist, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total, int key_bits,
                       uint32_t param, uint16_t* out, void* stream) {
  (void)n_total;
  if (n && !out) return -1;
  if (key_bits < 1 || key_bits > 16) return -1;
  if (dist < 0 || dist > FSG_CONST || dist == FSG_SORTEDSWAP) return -1;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t* T = nullptr;
  const uint32_t* G = nullptr;
  const uint16_t* perm = nullptr;
  if (dist == FSG_ZIPF || dist == FSG_GAUSS) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -3;
    std::lock_guard<std::mutex> lock(g_mu);
    DevTables& t = g_dev[dev];
    if (t.dist != dist || t.seed != seed) {
      uint64_t* hT = (uint64_t*)malloc(8 * kNumValues);
      uint32_t* hG = (uint32_t*)malloc(4 * kNumValues);
      uint16_t* hP = (uint16_t*)malloc(2 * kNumValues);
      if (!hT || !hG || !hP) return -2;
      int rc = host_tables(dist, seed, hT, hG, hP);
      if (rc) return rc;
      if (!t.T) {
        if (int e = cuda_rc(cudaMalloc(&t.T, 8 * kNumValues))) return e;
        if (int e = cuda_rc(cudaMalloc(&t.G, 4 * kNumValues))) return e;
        if (int e = cuda_rc(cudaMalloc(&t.perm, 2 * kNumValues))) return e;
      }
      // Synchronous copies: the tables must be in place before any kernel reads them.
      if (int e = cuda_rc(cudaMemcpy(t.T, hT, 8 * kNumValues, cudaMemcpyHostToDevice))) return e;
      if (int e = cuda_rc(cudaMemcpy(t.G, hG, 4 * kNumValues, cudaMemcpyHostToDevice))) return e;
      if (int e = cuda_rc(cudaMemcpy(t.perm, hP, 2 * kNumValues, cudaMemcpyHostToDevice))) return e;
      free(hT);
      free(hG);
      free(hP);
      t.dist = dist;
      t.seed = seed;
    }
    T = t.T;
    G = t.G;
    perm = t.perm;
  }
  const uint64_t ks = fsg_stream_key(seed, stream_for(dist));
  k_gen_u16<<<grid_for(n), 256, 0, s>>>(dist, ks, i0, n, key_bits, param, T, G, perm, out);
  return cuda_rc(cudaGetLastError());
}

int fsg_gen_u32_host(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint32_t* out) {
  if ((n && !out) || key_bits < 1 || key_bits > 32) return -1;
  const uint64_t ks = fsg_stream_key(seed, FSG_STREAM_U64);
  for (uint64_t j = 0; j < n; ++j) out[j] = (uint32_t)(fsg_draw_k(ks, i0 + j) >> (64 - key_bits));
  return 0;
}

int fsg_gen_u64_host(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint64_t* out) {
  if ((n && !out) || key_bits < 1 || key_bits > 64) return -1;
  const uint64_t ks = fsg_stream_key(seed, FSG_STREAM_U64);
  for (uint64_t j = 0; j < n; ++j) out[j] = fsg_draw_k(ks, i0 + j) >> (64 - key_bits);
  return 0;
}

int fsg_gen_u32_device(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint32_t* out, void* stream) {
  if ((n && !out) || key_bits < 1 || key_bits > 32) return -1;
  if (!n) return 0;
  k_gen_wide<uint32_t><<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      fsg_stream_key(seed, FSG_STREAM_U64), i0, n, key_bits, out);
  return cuda_rc(cudaGetLastError());
}

int fsg_gen_u64_device(uint64_t seed, uint64_t i0, uint64_t n, int key_bits, uint64_t* out, void* stream) {
  if ((n && !out) || key_bits < 1 || key_bits > 64) return -1;
  if (!n) return 0;
  k_gen_wide<uint64_t><<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      fsg_stream_key(seed, FSG_STREAM_U64), i0, n, key_bits, out);
  return cuda_rc(cudaGetLastError());
}

int fsg_iota_u32_host(uint64_t i0, uint64_t n, uint32_t* out) {
  if (n && !out) return -1;
  for (uint64_t j = 0; j < n; ++j) out[j] = (uint32_t)(i0 + j);
  return 0;
}

int fsg_iota_u32_device(uint64_t i0, uint64_t n, uint32_t* out, void* stream) {
  if (n && !out) return -1;
  if (!n) return 0;
  k_iota<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(i0, n, out);
  return cuda_rc(cudaGetLastError());
}

}  // extern "C"
