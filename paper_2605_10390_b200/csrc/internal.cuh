// internal.cuh — host-side helpers shared by the ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "fractalsort.h"

namespace fs {

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Temp layout of the u16 path (all offsets 256-byte aligned).  Nothing needs
// zeroing by the caller: the histogram kernel zeroes its spill and flags.
struct U16Layout {
  int grid = 1;
  size_t spill_off = 0, slice_tot_off = 0, partials_off = 0, prefix_off = 0, total = 0;
};
U16Layout u16_layout(uint64_t n, bool with_prefix);

fs_status fail(fs_status s, const char* fmt, ...);
fs_status cuda_fail(cudaError_t e, const char* where);
fs_status finish(cudaStream_t s, const char* where);
void clear_error();

// NVTX ranges (header-only nvtx3: free unless a profiler is attached): one range
// per public call, named after it, and inside it one range per phase of the
// call (opened at every phase boundary, see phase_event).
struct NvtxScope {
  explicit NvtxScope(const char* name);
  ~NvtxScope();
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};
#define FS_ENTRY()   \
  ::fs::clear_error(); \
  ::fs::NvtxScope fs_nvtx_scope_(__func__)
bool overlaps(const void* a, size_t an, const void* b, size_t bn);
// Records phase event i on stream s if fs_set_phase_events armed one (thread-local).
void phase_event(int i, cudaStream_t s);

}  // namespace fs
