// Phase timing of the product k_hist16 (included with -DFS_HIST_TRACE): per-CTA
// %globaltimer stamps at prologue / main loop end / flush end / grid sync /
// merge end / scan end, on 2^28 uniform keys.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFS_HIST_TRACE \
//        -I../../include -I../../paper_2605_10390_b200/csrc -o ht hist_trace.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2605_10390_b200/csrc/hist16.cu"

namespace fs {
const DeviceInfo& device_info() { static DeviceInfo d; if (!d.sm_count) cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, 0); return d; }
}
__device__ __forceinline__ uint64_t sm64(uint64_t z){z+=0x9E3779B97F4A7C15ull;z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
__global__ void gen(uint16_t* k, uint64_t n){ for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n;i+=(uint64_t)gridDim.x*blockDim.x) k[i]=(uint16_t)(sm64(i)>>48); }

int main(int argc, char** argv){
  setvbuf(stdout,NULL,_IONBF,0);
  uint64_t n=argc>1?strtoull(argv[1],nullptr,0):1ull<<28; uint16_t* k; uint32_t* part; unsigned long long *sp; uint64_t *st; uint32_t* rw; uint64_t* P;
  int G=fs::hist16_grid(n);
  cudaMalloc(&k,n*2); cudaMalloc(&part,(size_t)G*131072); cudaMalloc(&sp,(65536+32)*8); cudaMalloc(&st,129*8); cudaMalloc(&rw,1024); cudaMalloc(&P,65537*8);
  gen<<<1184,256>>>(k,n); cudaDeviceSynchronize();
  for(int rep=0;rep<4;rep++){
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e=fs::launch_hist16(k,n,part,sp,nullptr,0,0,P,st,G,0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b);
    if(e!=cudaSuccess){printf("launch error %s\n",cudaGetErrorString(e));return 1;}
    unsigned long long tr[256][8]; cudaMemcpyFromSymbol(tr, g_hist_trace, sizeof(tr));
    unsigned long long t0=~0ull; for(int c=0;c<G;c++) t0=std::min(t0,tr[c][0]);
    printf("rep %d: event %.1f us\n",rep,ms*1e3);
    const char* nm[7]={"start","prologue+sync","mainloop end","flush end","sync2","merge+scan end","static end(w0)"};
    for(int i=0;i<7;i++){ std::vector<double> v; for(int c=0;c<G;c++) v.push_back((tr[c][i]-t0)/1e3); std::sort(v.begin(),v.end());
      printf("  %-14s min %7.2f  med %7.2f  max %7.2f us\n",nm[i],v[0],v[v.size()/2],v.back()); }
    if(rep==3){ // per-CTA main-loop duration vs SM id
      printf("cta smid mainloop_us static_us\n");
      for(int c=0;c<G;c++) printf("%d %llu %.2f %.2f\n", c, tr[c][7], (tr[c][2]-tr[c][1])/1e3, (tr[c][6]-tr[c][1])/1e3);
    }
  }
  return 0;
}
