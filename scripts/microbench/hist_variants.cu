// Microbenchmark: variants of the per-SM packed-u16 SMEM-atomic histogram loop
// (stage 1 of hist16.cu) on 2^28 keys of several distributions.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hv hist_variants.cu && ./hv
// Prints time and keys/clk/SM per variant; checks each histogram against V0.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

constexpr int T = 1024;
constexpr uint32_t kHot = 0xC000C000u;

__device__ __forceinline__ uint64_t sm64(uint64_t z){z+=0x9E3779B97F4A7C15ull;z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
__global__ void gen(uint16_t* k, uint64_t n, int mode){
  for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n;i+=(uint64_t)gridDim.x*blockDim.x){
    uint64_t d=sm64(i); uint16_t v=(uint16_t)(d>>48);
    if(mode==1){ uint64_t u=d&0xFFFFF; if(u<207618) v=4242; else if(u<297000) v=777; else if(u<352000) v=31000; }  // ~20%/8.5%/5%
    if(mode==2) v=0xA5A5;
    if(mode==3) v=(uint16_t)((i*65536ull)/n);
    if(mode==4){ double u=((d>>11)+0.5)*(1.0/9007199254740992.0); double r=pow(u,-1.0/0.2); uint64_t rk = r>65536.0?65535:(uint64_t)r-1; v=(uint16_t)(sm64(rk*7919+13)>>48); }
    k[i]=v; }
}

__device__ __noinline__ void spill_word(uint32_t* sh, uint32_t w, unsigned long long* spill){
  uint32_t x=atomicExch(&sh[w],0u);
  if(x&0xFFFFu) atomicAdd(&spill[2*w],(unsigned long long)(x&0xFFFFu));
  if(x>>16) atomicAdd(&spill[2*w+1],(unsigned long long)(x>>16));
}
__device__ __forceinline__ void add_key(uint32_t* sh, uint32_t k, uint32_t cnt, unsigned long long* spill){
  uint32_t w=k>>1; uint32_t old=atomicAdd(&sh[w],(k&1u)?(cnt<<16):cnt); if(old&kHot) spill_word(sh,w,spill);
}
__device__ __forceinline__ bool all8_equal(const uint4& v){ return (v.x==v.y)&(v.y==v.z)&(v.z==v.w)&((v.x>>16)==(v.x&0xFFFFu)); }

// ---- V0: the product kernel's loop as of round 1 commit 46875d0
__device__ __forceinline__ void add8_v0(uint32_t* sh, const uint4& v, unsigned long long* spill){
  const uint32_t w[4]={v.x,v.y,v.z,v.w}; uint32_t old[8];
  #pragma unroll
  for(int j=0;j<4;++j){ uint32_t lo=w[j]&0xFFFFu, hi=w[j]>>16;
    old[2*j]=atomicAdd(&sh[lo>>1],(lo&1u)?0x10000u:1u); old[2*j+1]=atomicAdd(&sh[hi>>1],(hi&1u)?0x10000u:1u); }
  #pragma unroll
  for(int j=0;j<4;++j){ if(old[2*j]&kHot) spill_word(sh,(w[j]&0xFFFFu)>>1,spill); if(old[2*j+1]&kHot) spill_word(sh,w[j]>>17,spill); }
}
__device__ __forceinline__ void add8_agg(uint32_t* sh, const uint4& v, unsigned long long* spill){
  const bool eq=all8_equal(v); const uint32_t k0=v.x&0xFFFFu; const uint32_t l0=__shfl_sync(~0u,k0,0);
  const bool same=__all_sync(~0u, eq && k0==l0);
  if(same){ if((threadIdx.x&31)==0) add_key(sh,k0,256u,spill);} else if(eq) add_key(sh,k0,8u,spill); else add8_v0(sh,v,spill);
}

// ---- V1: returns OR-accumulated, one check per group; branch-light increments
__device__ __forceinline__ uint32_t add8_v1(uint32_t* sh, const uint4& v){
  const uint32_t w[4]={v.x,v.y,v.z,v.w}; uint32_t acc=0;
  char* base=reinterpret_cast<char*>(sh);
  #pragma unroll
  for(int j=0;j<4;++j){ const uint32_t x=w[j];
    const uint32_t alo=(x+x)&0x1FFFCu, ahi=(x>>15)&0x1FFFCu;              // byte offsets of words k>>1
    const uint32_t ilo=(x&1u)*0xFFFFu+1u, ihi=max(x&0x10000u,1u);         // 1 or 0x10000
    acc|=atomicAdd(reinterpret_cast<uint32_t*>(base+alo),ilo);
    acc|=atomicAdd(reinterpret_cast<uint32_t*>(base+ahi),ihi); }
  return acc;
}
__device__ __forceinline__ void recheck1(uint32_t* sh, const uint4 q, unsigned long long* spill){
  const uint32_t w[4]={q.x,q.y,q.z,q.w};
  #pragma unroll
  for(int j=0;j<4;++j){ uint32_t a=(w[j]&0xFFFFu)>>1, b=w[j]>>17;
    if(sh[a]&kHot) spill_word(sh,a,spill); if(sh[b]&kHot) spill_word(sh,b,spill); }
}
__device__ __forceinline__ uint32_t add8_match(uint32_t* sh, const uint4& v){
  const uint32_t w[4]={v.x,v.y,v.z,v.w}; uint32_t acc=0; const uint32_t lane=threadIdx.x&31;
  #pragma unroll
  for(int j=0;j<4;++j){
    #pragma unroll
    for(int e=0;e<2;++e){ const uint32_t k = e ? (w[j]>>16) : (w[j]&0xFFFFu);
      const uint32_t peers=__match_any_sync(~0u,k);
      const uint32_t leader=__ffs(peers)-1;
      if(lane==leader){ const uint32_t c=__popc(peers); acc|=atomicAdd(&sh[k>>1],(k&1u)?(c<<16):c); } } }
  return acc;
}
// hot-bin promotion: bins registered in hot[4] are counted in per-thread registers
__device__ __forceinline__ uint32_t add8_hot(uint32_t* sh, const uint4& v, const uint32_t h[4], uint32_t c[4]){
  const uint32_t w[4]={v.x,v.y,v.z,v.w}; uint32_t acc=0;
  #pragma unroll
  for(int j=0;j<4;++j){
    #pragma unroll
    for(int e=0;e<2;++e){ const uint32_t k = e ? (w[j]>>16) : (w[j]&0xFFFFu);
      const bool m0=k==h[0], m1=k==h[1], m2=k==h[2], m3=k==h[3];
      c[0]+=m0; c[1]+=m1; c[2]+=m2; c[3]+=m3;
      if(!(m0|m1|m2|m3)) acc|=atomicAdd(&sh[k>>1],(k&1u)?0x10000u:1u); } }
  return acc;
}
__device__ __forceinline__ void register_hot(uint32_t* hot, uint32_t* hot_any, uint32_t w, uint32_t x){
  // x: the exchanged word; register the hot half (or halves)
  #pragma unroll
  for(int e=0;e<2;++e){ const uint32_t half = e ? (x>>16) : (x&0xFFFFu); if(half < 0x4000u) continue;
    const uint32_t bin=2*w+e; bool present=false;
    for(int s=0;s<4;++s) present |= (hot[s]==bin);
    if(!present){ for(int s=0;s<4;++s){ if(atomicCAS(&hot[s],0xFFFFFFFFu,bin)==0xFFFFFFFFu){ atomicExch(hot_any,1u); break; } } } }
}
__device__ __forceinline__ void recheck_hot(uint32_t* sh, const uint4 q, unsigned long long* spill, uint32_t* hot, uint32_t* hot_any){
  const uint32_t w[4]={q.x,q.y,q.z,q.w};
  #pragma unroll
  for(int j=0;j<4;++j){
    #pragma unroll
    for(int e=0;e<2;++e){ const uint32_t a = e ? (w[j]>>17) : ((w[j]&0xFFFFu)>>1);
      if(sh[a]&kHot){ uint32_t x=atomicExch(&sh[a],0u);
        if(x&0xFFFFu) atomicAdd(&spill[2*a],(unsigned long long)(x&0xFFFFu));
        if(x>>16) atomicAdd(&spill[2*a+1],(unsigned long long)(x>>16));
        register_hot(hot,hot_any,a,x); } } }
}

template<int V,int U>
__global__ void __launch_bounds__(T,1) hist(const uint4* __restrict__ in, uint64_t n4, uint32_t* partials, unsigned long long* spill){
  extern __shared__ uint4 sm4[]; uint32_t* sh=reinterpret_cast<uint32_t*>(sm4);
  __shared__ uint32_t hot[4]; __shared__ uint32_t hot_any_s; uint32_t* hot_any=&hot_any_s;
  uint32_t hc[4]={0,0,0,0};
  for(int i=threadIdx.x;i<8192;i+=T) sm4[i]=make_uint4(0,0,0,0);
  if(threadIdx.x<4) hot[threadIdx.x]=0xFFFFFFFFu; if(threadIdx.x==0) hot_any_s=0;
  __syncthreads();
  const uint64_t stride=(uint64_t)gridDim.x*T; uint64_t i=blockIdx.x*(uint64_t)T+threadIdx.x;
  const uint64_t wt=31-(threadIdx.x&31);
  for(; i+wt+(U-1)*stride<n4; i+=U*stride){
    uint4 v[U];
    #pragma unroll
    for(int u=0;u<U;u++) v[u]=__ldcs(in+i+u*stride);
    if(V==0){
      bool runs=false;
      #pragma unroll
      for(int u=0;u<U;u++) runs|=all8_equal(v[u]);
      if(__any_sync(~0u,runs)){
        #pragma unroll
        for(int u=0;u<U;u++) add8_agg(sh,v[u],spill);
      } else {
        #pragma unroll
        for(int u=0;u<U;u++) add8_v0(sh,v[u],spill);
      }
    } else if(V==1 || V==2){
      const bool runs = V==1 ? all8_equal(v[0]) : false;
      if(V==1 && __any_sync(~0u,runs)){
        #pragma unroll
        for(int u=0;u<U;u++) add8_agg(sh,v[u],spill);
      } else {
        uint32_t acc=0;
        #pragma unroll
        for(int u=0;u<U;u++) acc|=add8_v1(sh,v[u]);
        if(acc&kHot){
          #pragma unroll
          for(int u=0;u<U;u++) recheck1(sh,v[u],spill);
        }
      }
    } else if(V==4){
      const bool runs = all8_equal(v[0]);
      if(__any_sync(~0u,runs)){
        #pragma unroll
        for(int u=0;u<U;u++) add8_agg(sh,v[u],spill);
      } else if(__any_sync(~0u, *hot_any != 0u)){
        const uint32_t h[4]={hot[0],hot[1],hot[2],hot[3]}; uint32_t acc=0;
        #pragma unroll
        for(int u=0;u<U;u++) acc|=add8_hot(sh,v[u],h,hc);
        if(acc&kHot){
          #pragma unroll
          for(int u=0;u<U;u++) recheck_hot(sh,v[u],spill,hot,hot_any);
        }
      } else {
        uint32_t acc=0;
        #pragma unroll
        for(int u=0;u<U;u++) acc|=add8_v1(sh,v[u]);
        if(acc&kHot){
          #pragma unroll
          for(int u=0;u<U;u++) recheck_hot(sh,v[u],spill,hot,hot_any);
        }
      }
    } else if(V==5){
      const bool runs = all8_equal(v[0]);
      if(__any_sync(~0u,runs)){
        #pragma unroll
        for(int u=0;u<U;u++) add8_agg(sh,v[u],spill);
      } else if(__any_sync(~0u, *hot_any != 0u)){
        uint32_t acc=0;
        #pragma unroll
        for(int u=0;u<U;u++) acc|=add8_match(sh,v[u]);
        if(acc&kHot){
          #pragma unroll
          for(int u=0;u<U;u++) recheck_hot(sh,v[u],spill,hot,hot_any);
        }
      } else {
        uint32_t acc=0;
        #pragma unroll
        for(int u=0;u<U;u++) acc|=add8_v1(sh,v[u]);
        if(acc&kHot){
          #pragma unroll
          for(int u=0;u<U;u++) recheck_hot(sh,v[u],spill,hot,hot_any);
        }
      }
    } else {  // V==3: no return values at all (unsafe: no overflow handling) -- lower bound
      #pragma unroll
      for(int u=0;u<U;u++){ const uint32_t w[4]={v[u].x,v[u].y,v[u].z,v[u].w};
        #pragma unroll
        for(int j=0;j<4;++j){ uint32_t x=w[j]; char* b=reinterpret_cast<char*>(sh);
          atomicAdd(reinterpret_cast<uint32_t*>(b+((x+x)&0x1FFFCu)),(x&1u)*0xFFFFu+1u);
          atomicAdd(reinterpret_cast<uint32_t*>(b+((x>>15)&0x1FFFCu)),max(x&0x10000u,1u)); } }
    }
  }
  for(; i<n4; i+=stride){ uint4 q=in[i]; add8_v0(sh,q,spill); }
  if(V==4){ // flush promoted counters: warp-reduce, one global atomic per warp per slot
    #pragma unroll
    for(int s2=0;s2<4;++s2){ uint32_t c=hc[s2]; for(int d=16;d;d>>=1) c+=__shfl_xor_sync(~0u,c,d);
      if((threadIdx.x&31)==0 && c) atomicAdd(&spill[hot[s2]],(unsigned long long)c); } }
  __syncthreads();
  uint4* p=reinterpret_cast<uint4*>(partials+(uint64_t)blockIdx.x*32768);
  for(int j=threadIdx.x;j<8192;j+=T) p[j]=sm4[j];
}

template<int U>
__global__ void __launch_bounds__(T,1) hist_pf(const uint4* __restrict__ in, uint64_t n4, uint32_t* partials, unsigned long long* spill){
  extern __shared__ uint4 sm4[]; uint32_t* sh=reinterpret_cast<uint32_t*>(sm4);
  for(int i=threadIdx.x;i<8192;i+=T) sm4[i]=make_uint4(0,0,0,0);
  __syncthreads();
  const uint64_t stride=(uint64_t)gridDim.x*T; uint64_t i=blockIdx.x*(uint64_t)T+threadIdx.x;
  const uint64_t wt=31-(threadIdx.x&31);
  uint4 nx[U];
  bool have = i+wt+(U-1)*stride<n4;
  if(have){
    #pragma unroll
    for(int u=0;u<U;u++) nx[u]=__ldcs(in+i+u*stride);
  }
  while(have){
    uint4 v[U];
    #pragma unroll
    for(int u=0;u<U;u++) v[u]=nx[u];
    const uint64_t j=i+U*stride;
    const bool more = j+wt+(U-1)*stride<n4;
    if(more){
      #pragma unroll
      for(int u=0;u<U;u++) nx[u]=__ldcs(in+j+u*stride);
    }
    uint32_t acc=0;
    #pragma unroll
    for(int u=0;u<U;u++) acc|=add8_v1(sh,v[u]);
    if(acc&kHot){
      #pragma unroll
      for(int u=0;u<U;u++) recheck1(sh,v[u],spill);
    }
    i=j; have=more;
  }
  for(; i<n4; i+=stride){ uint4 q=in[i]; add8_v0(sh,q,spill); }
  __syncthreads();
  uint4* p=reinterpret_cast<uint4*>(partials+(uint64_t)blockIdx.x*32768);
  for(int j=threadIdx.x;j<8192;j+=T) p[j]=sm4[j];
}

// total per bin = sum over CTAs + spill
__global__ void reduce(const uint32_t* partials, int G, const unsigned long long* spill, unsigned long long* C){
  int b=blockIdx.x*blockDim.x+threadIdx.x; if(b>=65536) return;
  unsigned long long c=spill[b];
  for(int g=0;g<G;g++){ uint32_t w=partials[(uint64_t)g*32768+(b>>1)]; c+=(b&1)?(w>>16):(w&0xFFFFu); }
  C[b]=c;
}

template<int U> float run_pf(const uint4* in, uint64_t n4, uint32_t* part, unsigned long long* sp, unsigned long long* C, int G, std::vector<unsigned long long>& hostC){
  auto k=hist_pf<U>; cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,131072);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best=1e9;
  for(int r=0;r<6;r++){
    cudaMemset(sp,0,65536*8);
    cudaEventRecord(a); k<<<G,T,131072>>>(in,n4,part,sp); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); if(r>0&&ms<best) best=ms;
  }
  reduce<<<256,256>>>(part,G,sp,C); hostC.resize(65536); cudaMemcpy(hostC.data(),C,65536*8,cudaMemcpyDeviceToHost);
  return best;
}
template<int V,int U> float run(const uint4* in, uint64_t n4, uint32_t* part, unsigned long long* sp, unsigned long long* C, int G, std::vector<unsigned long long>& hostC){
  auto k=hist<V,U>; cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,131072);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best=1e9;
  for(int r=0;r<6;r++){
    cudaMemset(sp,0,65536*8);
    cudaEventRecord(a); k<<<G,T,131072>>>(in,n4,part,sp); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); if(r>0&&ms<best) best=ms;
  }
  reduce<<<256,256>>>(part,G,sp,C); hostC.resize(65536); cudaMemcpy(hostC.data(),C,65536*8,cudaMemcpyDeviceToHost);
  return best;
}

int main(){ setvbuf(stdout,NULL,_IONBF,0);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  uint64_t n=1ull<<28; uint16_t* k; uint32_t* part; unsigned long long *sp,*C;
  CK(cudaMalloc(&k,n*2)); CK(cudaMalloc(&part,(size_t)sms*131072)); CK(cudaMalloc(&sp,65536*8)); CK(cudaMalloc(&C,65536*8));
  const char* names[5]={"uniform","hot3","allequal","sorted","zipf"};
  for(int mode=0;mode<5;mode++){
    gen<<<sms*8,512>>>(k,n,mode); CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> c0,c1,c2;
    float t0=run<0,4>((uint4*)k,n/8,part,sp,C,sms,c0);
    float t1=run<1,4>((uint4*)k,n/8,part,sp,C,sms,c1);
    float t2=run<1,2>((uint4*)k,n/8,part,sp,C,sms,c2);
    std::vector<unsigned long long> cx; float t3=mode==0?run<2,4>((uint4*)k,n/8,part,sp,C,sms,cx):0;
    float t4=mode==0?run<3,4>((uint4*)k,n/8,part,sp,C,sms,cx):0;
    std::vector<unsigned long long> c5; float t5=run<4,4>((uint4*)k,n/8,part,sp,C,sms,c5);
    std::vector<unsigned long long> c6; float t6=run<4,2>((uint4*)k,n/8,part,sp,C,sms,c6);
    if(mode==0||mode==4){ std::vector<unsigned long long> p1,p2; float a1=run_pf<2>((uint4*)k,n/8,part,sp,C,sms,p1); float a2=run_pf<1>((uint4*)k,n/8,part,sp,C,sms,p2);
      printf("   PF U2 %.1f us (%s)  PF U1 %.1f us (%s)\n", a1*1e3, p1==c0?"ok":"MISMATCH", a2*1e3, p2==c0?"ok":"MISMATCH"); }
    std::vector<unsigned long long> c7; float t7=run<5,4>((uint4*)k,n/8,part,sp,C,sms,c7);
    std::vector<unsigned long long> c8; float t8=run<5,2>((uint4*)k,n/8,part,sp,C,sms,c8);
    printf("   V5(match when hot) U4 %.1f us (%s)  U2 %.1f us (%s)\n", t7*1e3, c7==c0?"ok":"MISMATCH", t8*1e3, c8==c0?"ok":"MISMATCH");
    printf("   V4(hot promotion) U4 %.1f us (%s)  U2 %.1f us (%s)\n", t5*1e3, c5==c0?"ok":"MISMATCH", t6*1e3, c6==c0?"ok":"MISMATCH");
    bool ok1=c0==c1, ok2=c0==c2; unsigned long long tot=0; for(auto x:c0) tot+=x;
    printf("[%s] total=%llu  V0 %.1f us | V1U4 %.1f us (%s) | V1U2 %.1f us (%s) | V2(no-runs)U4 %.1f | V3(red,unsafe) %.1f\n",
      names[mode],tot,t0*1e3,t1*1e3,ok1?"ok":"MISMATCH",t2*1e3,ok2?"ok":"MISMATCH",t3*1e3,t4*1e3);
  }
  CK(cudaGetLastError()); return 0;
}
