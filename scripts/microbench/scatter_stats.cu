// Lookback statistics of k_scatter on c5 (2^29 pairs), per pass mode: digit-threads
// x tiles that looked back, rounds of 8 loads, polls of unpublished words, and
// how often the immediate predecessor already held the inclusive prefix.
// Build: see scripts/microbench/README (objects compiled with -DFS_SCATTER_STATS -dc).
#include <cstdio>
#include <cuda_runtime.h>
#include "fractalsort.h"
extern __device__ unsigned long long g_scatter_stats[3][4];
extern __device__ unsigned long long g_scatter_phase[3][8];
extern __device__ unsigned long long g_local_phase[8];
__device__ __forceinline__ unsigned long long sm64(unsigned long long z){z+=0x9E3779B97F4A7C15ull;z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
__global__ void gen(unsigned long long* k, unsigned* v, unsigned long long n){ for(unsigned long long i=blockIdx.x*(unsigned long long)blockDim.x+threadIdx.x;i<n;i+=(unsigned long long)gridDim.x*blockDim.x){k[i]=sm64(i);v[i]=(unsigned)i;} }
int main(){
  const unsigned long long n = 1ull << 29;
  unsigned long long *k,*ko; unsigned *v,*vo; void* t;
  size_t tb = fs_sort_pairs_u64_u32_temp_bytes(n, 64);
  cudaMalloc(&k,n*8); cudaMalloc(&ko,n*8); cudaMalloc(&v,n*4); cudaMalloc(&vo,n*4); cudaMalloc(&t,tb);
  gen<<<1184,256>>>(k,v,n); cudaDeviceSynchronize();
  for (int rep=0; rep<2; ++rep) {
    unsigned long long z[3][4] = {}, ph[3][8] = {};
    cudaMemcpyToSymbol(g_scatter_stats, z, sizeof(z));
    cudaMemcpyToSymbol(g_scatter_phase, ph, sizeof(ph));
    unsigned long long lp[8] = {};
    cudaMemcpyToSymbol(g_local_phase, lp, sizeof(lp));
    fs_status s = fs_sort_pairs_u64_u32((const uint64_t*)k, v, (uint64_t*)ko, vo, n, 64, t, tb, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z, g_scatter_stats, sizeof(z));
    cudaMemcpyFromSymbol(ph, g_scatter_phase, sizeof(ph));
    cudaMemcpyFromSymbol(lp, g_local_phase, sizeof(lp));
    {
      const char* ln[6] = {"load+count", "scan", "scatter", "rank+keys", "slow", "values"};
      unsigned long long tot = 0; for (int i = 0; i < 6; ++i) tot += lp[i];
      printf("  local sort phases:"); for (int i = 0; i < 6; ++i) printf(" %s %.1f", ln[i], 100.0 * lp[i] / tot); printf("\n");
    }
    const char* nm[7] = {"fetch+wait", "items+rank+bar", "counts+scan+offsets", "reorder", "lookback+bar", "scatter", "end-bar"};
    for (int m = 1; m < 3; ++m) {
      unsigned long long tot = 0; for (int i = 0; i < 7; ++i) tot += ph[m][i];
      printf("  mode %d phases (%% of thread-0 cycles):", m);
      for (int i = 0; i < 7; ++i) printf(" %s %.1f", nm[i], 100.0 * ph[m][i] / tot);
      printf("\n");
    }
    printf("rep %d status %d\n", rep, (int)s);
    for (int m = 1; m < 3; ++m)
      printf("  mode %d: lookbacks %llu  rounds/lookback %.3f  polls/lookback %.3f  inc-at-first %.3f\n", m, z[m][0],
             (double)z[m][1] / z[m][0], (double)z[m][2] / z[m][0], (double)z[m][3] / z[m][0]);
  }
  return 0;
}
