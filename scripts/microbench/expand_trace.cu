// Per-CTA timeline of the product k_expand16 (included with -DFS_EXPAND_TRACE) on
// the c2 prefix (2^28 uniform keys): %globaltimer at start, after the setup
// (search + staging), after the last store; prints the distribution of setup and
// store durations per wave and the number of CTAs storing over time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFS_EXPAND_TRACE \
//        -I../../include -I../../paper_2605_10390_b200/csrc -o expand_trace expand_trace.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cstring>
#include "../../paper_2605_10390_b200/csrc/expand16.cu"

namespace fs {
const DeviceInfo& device_info() { static DeviceInfo d; if (!d.sm_count) cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, 0); return d; }
}
// uniform-like prefix: C[v] = n / 65536 (two-level form: slice-local L and slice totals)
__global__ void mkprefix(uint64_t* L, uint64_t* tot, uint64_t per) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < 65536) L[v] = (uint64_t)(v & 511) * per;
  if (v < 128) tot[v] = per * 512;
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1ull << 28);
  uint64_t *L, *tot; uint16_t* out;
  cudaMalloc(&L, 65536 * 8); cudaMalloc(&tot, 128 * 8); cudaMalloc(&out, n * 2);
  const char* dist = argc > 2 ? argv[2] : "uniform";
  if (!strcmp(dist, "uniform")) {
    mkprefix<<<256, 256>>>(L, tot, n / 65536);
  } else {  // gauss (mean 32768, sd 1024) or zipf (s = 1.2, values permuted): expected counts
    std::vector<double> w(65536);
    if (!strcmp(dist, "gauss")) {
      for (int v = 0; v < 65536; ++v) w[v] = 0.5 * (erf((v + 0.5 - 32768) / 1024 / sqrt(2.0)) - erf((v - 0.5 - 32768) / 1024 / sqrt(2.0)));
    } else {
      std::vector<int> perm(65536);
      for (int v = 0; v < 65536; ++v) perm[v] = v;
      uint64_t x = 88172645463325252ull;
      for (int v = 65535; v > 0; --v) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; std::swap(perm[v], perm[x % (v + 1)]); }
      for (int r = 0; r < 65536; ++r) w[perm[r]] = pow(r + 1.0, -1.2);
    }
    double sw = 0; for (double y : w) sw += y;
    std::vector<uint64_t> C(65536), hL(65536), ht(128, 0);
    uint64_t tot_c = 0;
    for (int v = 0; v < 65536; ++v) { C[v] = (uint64_t)(w[v] / sw * n); tot_c += C[v]; }
    C[32768] += n - tot_c;
    for (int s = 0; s < 128; ++s) { uint64_t run = 0; for (int j = 0; j < 512; ++j) { hL[s * 512 + j] = run; run += C[s * 512 + j]; } ht[s] = run; }
    cudaMemcpy(L, hL.data(), 65536 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(tot, ht.data(), 128 * 8, cudaMemcpyHostToDevice);
  }
  cudaDeviceSynchronize();
  static unsigned long long tr[1 << 16][4];
  for (int rep = 0; rep < 4; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = fs::launch_expand16_two_level(L, tot, 0, n, out, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return 1; }
    const int G = (int)std::min<uint64_t>((n / 8 + 4095) / 4096, 1 << 16);
    cudaMemcpyFromSymbol(tr, g_expand_trace, sizeof(unsigned long long) * 4 * G);
    unsigned long long t0 = ~0ull, tend = 0;
    for (int c = 0; c < G; c++) { t0 = std::min(t0, tr[c][0]); tend = std::max(tend, tr[c][2]); }
    std::vector<double> setup, store, start;
    for (int c = 0; c < G; c++) { setup.push_back((tr[c][1] - tr[c][0]) / 1e3); store.push_back((tr[c][2] - tr[c][1]) / 1e3); start.push_back((tr[c][0] - t0) / 1e3); }
    auto q = [](std::vector<double> v, double f) { std::sort(v.begin(), v.end()); return v[(size_t)(f * (v.size() - 1))]; };
    printf("rep %d: event %.1f us, first start -> last end %.1f us, %d CTAs\n", rep, ms * 1e3, (tend - t0) / 1e3, G);
    printf("  setup us  p10 %.2f p50 %.2f p90 %.2f max %.2f\n", q(setup, .1), q(setup, .5), q(setup, .9), q(setup, 1));
    printf("  store us  p10 %.2f p50 %.2f p90 %.2f max %.2f\n", q(store, .1), q(store, .5), q(store, .9), q(store, 1));
    if (rep == 3) {  // slowest CTAs, and CTAs in setup / storing per microsecond
      std::vector<std::pair<double, int>> tot_t;
      for (int c = 0; c < G; c++) tot_t.push_back({(tr[c][2] - tr[c][0]) / 1e3, c});
      std::sort(tot_t.rbegin(), tot_t.rend());
      printf("  slowest CTAs (us, tile):");
      for (int i = 0; i < 12; ++i) printf(" %.1f@%d", tot_t[i].first, tot_t[i].second);
      printf("\n");
      const int T = (int)((tend - t0) / 1000) + 1;
      std::vector<int> in_setup(T, 0), storing(T, 0);
      for (int c = 0; c < G; c++) {
        for (int t = (int)((tr[c][0] - t0) / 1000); t <= (int)((tr[c][1] - t0) / 1000) && t < T; ++t) in_setup[t]++;
        for (int t = (int)((tr[c][1] - t0) / 1000); t <= (int)((tr[c][2] - t0) / 1000) && t < T; ++t) storing[t]++;
      }
      printf("  us: CTAs in setup / storing\n");
      for (int t = 0; t < T; ++t) printf("  %3d %5d %5d\n", t, in_setup[t], storing[t]);
    }
  }
  return 0;
}
