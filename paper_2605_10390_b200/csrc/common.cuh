// common.cuh — small device helpers shared by the sm_100a kernels of libfractalsort.so.
// (Product code: nothing here is shared with oracle/ or datagen/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fractalsort.h"

#define FS_DEVINL __device__ __forceinline__

namespace fs {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xFFFFFFFFu;

// 128-bit streaming load of data read exactly once (ld.global.cs: evict-first).
FS_DEVINL uint4 ld_stream_v4(const uint4* p) { return __ldcs(p); }

// 128-bit streaming store (written once, not re-read by this kernel).
#ifndef FS_STORE_FLAVOR  // scripts/microbench: 0 .cs, 1 plain (write-back), 2 .L1::no_allocate
#define FS_STORE_FLAVOR 0
#endif
FS_DEVINL void st_stream_v4(uint4* p, uint4 v) {
#if FS_STORE_FLAVOR == 1
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
#elif FS_STORE_FLAVOR == 2
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
#else
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
#endif
}

// 64-bit status words of the decoupled lookbacks.  A status word carries its own
// value (flag | count), and nothing else is published through it, so relaxed
// GPU-scope accesses suffice.  (On sm_100a ld.acquire.gpu compiles to
// LDG.STRONG + CCTL.IVALL -- an L1 invalidate per poll -- and st.release to a
// MEMBAR; both were the top stalls of the first onesweep.)
FS_DEVINL void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
FS_DEVINL unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
FS_DEVINL void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
FS_DEVINL unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

FS_DEVINL uint32_t lane_id() { return threadIdx.x & 31u; }
FS_DEVINL uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Inclusive warp scan (Kogge-Stone over shuffles).
template <typename T>
FS_DEVINL T warp_inclusive_scan(T x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(kFull, x, d);
    if ((int)lane_id() >= d) x += y;
  }
  return x;
}

template <typename T>
FS_DEVINL T warp_sum(T x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}

// Decoupled-lookback status word: [63:62] flag, [61:0] value.
constexpr unsigned long long kFlagAggregate = 1ull << 62;
constexpr unsigned long long kFlagInclusive = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

}  // namespace fs
