// nvls.cu — the cross-GPU histogram merge through NVSwitch multicast (NVLS):
// SURVEY.md §8(f) NEXT-2 "NVLS all-reduce of the histogram", §8(e) row a3
// across GPUs.
//
// What it computes: dst[i] = sum over the G ranks of src_r[i], i < count — the
// Global Histogram Update of PAPER.md:91-92 (§III.B: worker histograms merged
// into one global structure) taken across GPUs.  The summed arrays are the
// per-rank histograms, or the sort's two-level prefix (slice-local exclusive
// prefixes + slice totals), which is linear in the counts, so its sum over
// ranks is the prefix of the summed histogram (dist.py mode "N").
//
// B200 design: every rank's src_r is its own physical memory bound into ONE
// multicast object (cuMulticastCreate / cuMulticastBindMem, set up by dist.py
// through the driver API).  A load from the multicast address with
// multimem.ld_reduce.add is answered by the NVSwitch, which reads the word
// from every bound GPU and returns the sum: one-shot all-reduce, no staging
// buffer, no NCCL kernel, no second copy.  The same kernel carries the
// cross-GPU barrier the reduction needs: CTA 0 arrives with
// multimem.red.release.sys (+1 on a flag word in every rank's copy), and every
// CTA waits on its local copy of the flag with ld.acquire.sys until all G
// ranks arrived for this call (target = G x calls so far), so no rank reads
// before every rank's src_r is complete.  Callers alternate two src halves by
// call parity: a rank can reach call k + 2's writes only after every rank
// arrived at call k + 1, i.e. finished reading call k.
#include "common.cuh"
#include "internal.cuh"

namespace fs {
namespace {

constexpr int kThreads = 256;

FS_DEVINL uint64_t mc_ld_reduce_add_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

FS_DEVINL void mc_red_release_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

FS_DEVINL uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

FS_DEVINL uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kThreads)
    k_allreduce_mc(const uint64_t* __restrict__ src_mc, uint64_t* __restrict__ dst, uint64_t count,
                   uint32_t* flag_mc, const uint32_t* flag_local, uint32_t target, uint64_t timeout_ns,
                   uint32_t* timed_out) {
  __shared__ uint32_t s_give_up;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) mc_red_release_add_u32(flag_mc, 1u);
    // wrap-safe wait: every rank adds exactly G per call, so flag - target is a
    // small negative number until all have arrived.  A rank that never arrives
    // (a peer failed) must not hang this one: after timeout_ns the CTA gives up
    // and reports it in *timed_out (dst is then not written).
    const uint64_t t0 = globaltimer_ns();
    uint32_t give_up = 0;
    while ((int32_t)(ld_acquire_sys_u32(flag_local) - target) < 0) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > timeout_ns) {
        give_up = 1;
        atomicExch(timed_out, 1u);
        break;
      }
    }
    s_give_up = give_up;
  }
  __syncthreads();
  if (s_give_up) return;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < count; i += stride)
    dst[i] = mc_ld_reduce_add_u64(src_mc + i);
}

}  // namespace
}  // namespace fs

using namespace fs;

extern "C" fs_status fs_allreduce_multicast_u64(const uint64_t* src_mc, uint64_t* dst, uint64_t count,
                                                uint32_t* flag_mc, const uint32_t* flag_local, uint32_t target,
                                                uint64_t timeout_ns, uint32_t* timed_out, fs_stream_t stream) {
  FS_ENTRY();
  if (!flag_mc || !flag_local || !timed_out) return fail(FS_ERR_INVALID_ARGUMENT, "NULL flag pointer");
  if ((uintptr_t)timed_out & 3) return fail(FS_ERR_INVALID_ARGUMENT, "timed_out not 4-byte aligned");
  if (((uintptr_t)flag_mc | (uintptr_t)flag_local) & 3) return fail(FS_ERR_INVALID_ARGUMENT, "flag not 4-byte aligned");
  if (count > 0 && (!src_mc || !dst)) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with count > 0");
  if (((uintptr_t)src_mc | (uintptr_t)dst) & 7) return fail(FS_ERR_INVALID_ARGUMENT, "arrays not 8-byte aligned");
  if (count > 0 && overlaps(src_mc, count * 8, dst, count * 8))
    return fail(FS_ERR_INVALID_ARGUMENT, "src_mc and dst overlap");
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "fs_allreduce_multicast_u64: device query");
  // at most one CTA per SM; a CTA's wait depends only on the other ranks' CTA 0,
  // which arrives before it waits, so no co-residency is assumed
  const uint64_t want = (count + kThreads * 4 - 1) / (kThreads * 4);
  const unsigned grid = (unsigned)(want < 1 ? 1 : (want > (uint64_t)sms ? (uint64_t)sms : want));
  k_allreduce_mc<<<grid, kThreads, 0, s>>>(src_mc, dst, count, flag_mc, flag_local, target,
                                           timeout_ns ? timeout_ns : ~0ull, timed_out);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fs_allreduce_multicast_u64");
  return finish(s, "fs_allreduce_multicast_u64");
}
