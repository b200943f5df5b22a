// abi.cu — the C ABI of libfractalsort.so (include/fractalsort.h): argument
// validation, temp sizing and layout, dispatch to the kernels, error reporting.
// No allocation on the hot path; the only state is the per-device attribute cache.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "fractalsort.h"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {

// ------------------------------------------------------------------ errors
namespace {
thread_local char g_err[512] = "";
thread_local void* const* g_events = nullptr;
thread_local int g_nevents = 0;
thread_local int g_nvtx_depth = 0;         // public calls in progress on this thread (nesting)
thread_local bool g_nvtx_phase_open = false;
const char* const kPhaseNames[] = {"phase 0", "phase 1", "phase 2",  "phase 3",  "phase 4",  "phase 5",
                                   "phase 6", "phase 7", "phase 8",  "phase 9",  "phase 10", "phase 11",
                                   "phase 12", "phase 13", "phase 14", "phase 15", "phase 16"};
}  // namespace

NvtxScope::NvtxScope(const char* name) {
  if (g_nvtx_depth++ == 0) g_nvtx_phase_open = false;
  nvtxRangePushA(name);
}

NvtxScope::~NvtxScope() {
  if (g_nvtx_depth == 1 && g_nvtx_phase_open) {
    nvtxRangePop();
    g_nvtx_phase_open = false;
  }
  nvtxRangePop();
  --g_nvtx_depth;
}

void phase_event(int i, cudaStream_t s) {
  if (g_events && i >= 0 && i < g_nevents && g_events[i]) cudaEventRecord((cudaEvent_t)g_events[i], s);
  if (g_nvtx_depth == 1 && i >= 0 && i < (int)(sizeof(kPhaseNames) / sizeof(kPhaseNames[0]))) {
    if (g_nvtx_phase_open) nvtxRangePop();
    nvtxRangePushA(kPhaseNames[i]);
    g_nvtx_phase_open = true;
  }
}

fs_status fail(fs_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

fs_status cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? FS_ERR_OUT_OF_MEMORY : FS_ERR_CUDA, "%s: %s (%s)", where,
              cudaGetErrorName(e), cudaGetErrorString(e));
}

void clear_error() { g_err[0] = 0; }

bool sync_check_enabled() {
  static const bool on = [] {
    const char* v = getenv("FS_SYNC_CHECK");
    return v && v[0] && v[0] != '0';
  }();
  return on;
}

fs_status finish(cudaStream_t s, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, where);
  if (sync_check_enabled()) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, where);
  }
  return FS_OK;
}

// ------------------------------------------------------------ device cache
namespace {
constexpr int kMaxDevices = 64;
DeviceInfo g_info[kMaxDevices];
std::once_flag g_once[kMaxDevices];
}  // namespace

const DeviceInfo& device_info() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  std::call_once(g_once[dev], [dev] {
    DeviceInfo& d = g_info[dev];
    d.device = dev;
    if (cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) d.sm_count = 148;
    cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, dev);
    cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaGetLastError();  // attribute queries without a GPU must not poison later calls
  });
  return g_info[dev];
}

// ------------------------------------------------------------ temp layouts
U16Layout u16_layout(uint64_t n, bool with_prefix) {
  U16Layout L;
  L.grid = hist16_grid(n);
  size_t off = 0;
  L.spill_off = off;  // spill u64[65536], then the dynamic-work counter (kernels.cuh kHistSpillWords)
  off = align_up(off + sizeof(uint64_t) * kHistSpillWords);
  L.slice_tot_off = off;
  off = align_up(off + sizeof(uint64_t) * kHistSlices);
  L.partials_off = off;
  // the one-cluster sort (small16.cu) needs 16 partial rows whatever n
  const size_t rows = (with_prefix && n <= small16_max_n() && L.grid < 16) ? 16 : (size_t)L.grid;
  off = align_up(off + sizeof(uint32_t) * kHistWords * rows);
  L.prefix_off = off;
  if (with_prefix) off = align_up(off + sizeof(uint64_t) * (kHistBins + 1));
  L.total = off;
  return L;
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return an && bn && pa < pb + bn && pb < pa + an;
}

}  // namespace fs

using namespace fs;

extern "C" {

const char* fs_status_string(fs_status s) {
  switch (s) {
    case FS_OK: return "FS_OK";
    case FS_ERR_INVALID_ARGUMENT: return "FS_ERR_INVALID_ARGUMENT";
    case FS_ERR_CUDA: return "FS_ERR_CUDA";
    case FS_ERR_OUT_OF_MEMORY: return "FS_ERR_OUT_OF_MEMORY";
    case FS_ERR_UNSUPPORTED: return "FS_ERR_UNSUPPORTED";
  }
  return "FS_UNKNOWN_STATUS";
}

const char* fs_last_error_message(void) { return g_err; }

int fs_version(void) { return (1 << 16) | 0; }

fs_status fs_set_phase_events(void* const* events, int count) {
  g_events = count > 0 ? events : nullptr;
  g_nevents = events ? count : 0;
  return FS_OK;
}

size_t fs_sort_keys_u16_temp_bytes(uint64_t n) { return u16_layout(n, true).total; }
size_t fs_histogram_u16_temp_bytes(uint64_t n) { return u16_layout(n, false).total; }
size_t fs_exclusive_scan_u64_temp_bytes(uint64_t nbins) {
  return align_up(sizeof(uint64_t) * scan_tiles(nbins ? nbins : 1)) + 256;
}
size_t fs_sort_keys_u32_temp_bytes(uint64_t n, int key_bits) { return wide_temp_bytes(n, 4, key_bits, false); }
size_t fs_sort_keys_u64_temp_bytes(uint64_t n, int key_bits) { return wide_temp_bytes(n, 8, key_bits, false); }
size_t fs_sort_pairs_u64_u32_temp_bytes(uint64_t n, int key_bits) {
  return wide_temp_bytes(n, 8, key_bits, true);
}

fs_status fs_sort_keys_u16(const uint16_t* keys_in, uint16_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (key_bits < 0 || key_bits > 16) return fail(FS_ERR_INVALID_ARGUMENT, "key_bits %d not in 0..16", key_bits);
  if (n == 0) return FS_OK;
  if (!keys_in || !keys_out || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  if (((uintptr_t)keys_in | (uintptr_t)keys_out) & 1)
    return fail(FS_ERR_INVALID_ARGUMENT, "keys not 2-byte aligned");
  const U16Layout L = u16_layout(n, true);
  if (temp_bytes < L.total)
    return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, L.total);
  if (keys_in != keys_out && overlaps(keys_in, 2 * n, keys_out, 2 * n))
    return fail(FS_ERR_INVALID_ARGUMENT, "keys_in and keys_out partially overlap");
  if (overlaps(temp, L.total, keys_in, 2 * n) || overlaps(temp, L.total, keys_out, 2 * n))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp overlaps the keys");
  cudaStream_t s = (cudaStream_t)stream;
  char* t = (char*)temp;
  auto* spill = (unsigned long long*)(t + L.spill_off);
  auto* slice_tot = (uint64_t*)(t + L.slice_tot_off);
  auto* partials = (uint32_t*)(t + L.partials_off);
  auto* prefix = (uint64_t*)(t + L.prefix_off);
  phase_event(0, s);
  phase_event(1, s);
  cudaError_t e;
  if (n <= small16_max_n()) {  // one cluster launch: every stage on chip
    if ((e = launch_sort16_small(keys_in, n, keys_out, spill, partials, s)) != cudaSuccess)
      return cuda_fail(e, "fs_sort_keys_u16: sort16_small (one-cluster sort)");
    phase_event(2, s);
    phase_event(3, s);
    return finish(s, "fs_sort_keys_u16");
  }
  if ((e = launch_hist16(keys_in, n, partials, spill, nullptr, 0, 0, prefix, slice_tot, L.grid, s)) !=
      cudaSuccess)
    return cuda_fail(e, "fs_sort_keys_u16: hist16 (histogram + merge + scan)");
  phase_event(2, s);
  if ((e = launch_expand16_two_level(prefix, slice_tot, 0, n, keys_out, s)) != cudaSuccess)
    return cuda_fail(e, "fs_sort_keys_u16: expand16");
  phase_event(3, s);
  return finish(s, "fs_sort_keys_u16");
}

fs_status fs_histogram_u16(const uint16_t* keys, uint64_t n, int key_bits, uint64_t* hist, int accumulate,
                           void* temp, size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (key_bits < 0 || key_bits > 16) return fail(FS_ERR_INVALID_ARGUMENT, "key_bits %d not in 0..16", key_bits);
  if (!hist) return fail(FS_ERR_INVALID_ARGUMENT, "hist is NULL");
  const uint64_t nb = (uint64_t)1 << (key_bits ? key_bits : 16);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (accumulate) return FS_OK;
    cudaError_t e = cudaMemsetAsync(hist, 0, nb * sizeof(uint64_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "fs_histogram_u16: memset hist");
    return finish(s, "fs_histogram_u16");
  }
  if (!keys || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  if ((uintptr_t)keys & 1) return fail(FS_ERR_INVALID_ARGUMENT, "keys not 2-byte aligned");
  const U16Layout L = u16_layout(n, false);
  if (temp_bytes < L.total)
    return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, L.total);
  if (overlaps(temp, L.total, hist, nb * 8) || overlaps(temp, L.total, keys, 2 * n))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp overlaps keys or hist");
  char* t = (char*)temp;
  auto* spill = (unsigned long long*)(t + L.spill_off);
  auto* partials = (uint32_t*)(t + L.partials_off);
  cudaError_t e;
  if ((e = launch_hist16(keys, n, partials, spill, hist, nb, accumulate ? 1 : 0, nullptr, nullptr, L.grid, s)) !=
      cudaSuccess)
    return cuda_fail(e, "fs_histogram_u16: hist16 (histogram + merge)");
  return finish(s, "fs_histogram_u16");
}

fs_status fs_histogram_prefix_u16(const uint16_t* keys, uint64_t n, uint64_t* prefix2, void* temp, size_t temp_bytes,
                                  fs_stream_t stream) {
  FS_ENTRY();
  if (!prefix2) return fail(FS_ERR_INVALID_ARGUMENT, "prefix2 is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(prefix2, 0, sizeof(uint64_t) * (kHistBins + kHistSlices), s);
    if (e != cudaSuccess) return cuda_fail(e, "fs_histogram_prefix_u16: memset");
    return finish(s, "fs_histogram_prefix_u16");
  }
  if (!keys || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  if ((uintptr_t)keys & 1) return fail(FS_ERR_INVALID_ARGUMENT, "keys not 2-byte aligned");
  const U16Layout L = u16_layout(n, false);
  if (temp_bytes < L.total)
    return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, L.total);
  const size_t pb = sizeof(uint64_t) * (kHistBins + kHistSlices);
  if (overlaps(temp, L.total, prefix2, pb) || overlaps(temp, L.total, keys, 2 * n) || overlaps(keys, 2 * n, prefix2, pb))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp, keys and prefix2 must not overlap");
  char* t = (char*)temp;
  cudaError_t e = launch_hist16(keys, n, (uint32_t*)(t + L.partials_off), (unsigned long long*)(t + L.spill_off),
                                nullptr, 0, 0, prefix2, prefix2 + kHistBins, L.grid, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_histogram_prefix_u16");
  return finish(s, "fs_histogram_prefix_u16");
}

fs_status fs_expand_prefix_u16(const uint64_t* prefix2, uint64_t out_begin, uint64_t out_end, uint16_t* out,
                               fs_stream_t stream) {
  FS_ENTRY();
  if (out_end < out_begin) return fail(FS_ERR_INVALID_ARGUMENT, "out_end < out_begin");
  if (out_end == out_begin) return FS_OK;
  if (!prefix2 || !out) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((uintptr_t)out & 1) return fail(FS_ERR_INVALID_ARGUMENT, "out not 2-byte aligned");
  if (overlaps(prefix2, sizeof(uint64_t) * (kHistBins + kHistSlices), out, 2 * (out_end - out_begin)))
    return fail(FS_ERR_INVALID_ARGUMENT, "prefix2 and out overlap");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_expand16_two_level(prefix2, prefix2 + kHistBins, out_begin, out_end, out, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_expand_prefix_u16");
  return finish(s, "fs_expand_prefix_u16");
}

fs_status fs_exclusive_scan_u64(const uint64_t* hist, uint64_t* prefix, uint64_t nbins, void* temp,
                                size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (nbins == 0 || nbins > (1ull << 32)) return fail(FS_ERR_INVALID_ARGUMENT, "nbins %llu not in 1..2^32",
                                                     (unsigned long long)nbins);
  if (!hist || !prefix || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  const size_t need = fs_exclusive_scan_u64_temp_bytes(nbins);
  if (temp_bytes < need) return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, need);
  if (overlaps(hist, nbins * 8, prefix, (nbins + 1) * 8))
    return fail(FS_ERR_INVALID_ARGUMENT, "hist and prefix overlap");
  if (overlaps(temp, need, hist, nbins * 8) || overlaps(temp, need, prefix, (nbins + 1) * 8))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp overlaps hist or prefix");
  cudaStream_t s = (cudaStream_t)stream;
  auto* status = (unsigned long long*)temp;
  auto* ticket = (uint32_t*)((char*)temp + align_up(sizeof(uint64_t) * scan_tiles(nbins)));
  cudaError_t e = cudaMemsetAsync(temp, 0, need, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_exclusive_scan_u64: memset");
  if ((e = launch_merge_scan(nullptr, 0, nullptr, hist, nbins, nullptr, 0, 0, prefix, status, ticket, s)) !=
      cudaSuccess)
    return cuda_fail(e, "fs_exclusive_scan_u64: scan");
  return finish(s, "fs_exclusive_scan_u64");
}

fs_status fs_expand_u16(const uint64_t* prefix, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                        uint16_t* out, fs_stream_t stream) {
  FS_ENTRY();
  if (nbins == 0 || nbins > 65536) return fail(FS_ERR_INVALID_ARGUMENT, "nbins %llu not in 1..65536",
                                              (unsigned long long)nbins);
  if (out_end < out_begin) return fail(FS_ERR_INVALID_ARGUMENT, "out_end < out_begin");
  if (out_end == out_begin) return FS_OK;
  if (!prefix || !out) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((uintptr_t)out & 1) return fail(FS_ERR_INVALID_ARGUMENT, "out not 2-byte aligned");
  if (overlaps(prefix, (nbins + 1) * 8, out, 2 * (out_end - out_begin)))
    return fail(FS_ERR_INVALID_ARGUMENT, "prefix and out overlap");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_expand16(prefix, nbins, out_begin, out_end, out, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_expand_u16");
  return finish(s, "fs_expand_u16");
}

fs_status fs_send_counts(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint64_t* send,
                         fs_stream_t stream) {
  FS_ENTRY();
  if (G < 1 || G > 1024 || g < 0 || g >= G) return fail(FS_ERR_INVALID_ARGUMENT, "bad G=%d g=%d", G, g);
  if (nbins == 0 || nbins > 65536) return fail(FS_ERR_INVALID_ARGUMENT, "nbins not in 1..65536");
  if (!hist_all || !send) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (overlaps(hist_all, (uint64_t)G * nbins * 8, send, (uint64_t)G * 8))
    return fail(FS_ERR_INVALID_ARGUMENT, "hist_all and send overlap");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_send_counts(hist_all, G, g, nbins, send, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_send_counts");
  return finish(s, "fs_send_counts");
}

fs_status fs_bound_u64(const uint64_t* sorted, uint64_t n, const uint64_t* queries, uint64_t q, int upper,
                       uint64_t* out, fs_stream_t stream) {
  FS_ENTRY();
  if (q == 0) return FS_OK;
  if (!queries || !out || (n && !sorted)) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (upper != 0 && upper != 1) return fail(FS_ERR_INVALID_ARGUMENT, "upper must be 0 or 1");
  if (overlaps(queries, q * 8, out, q * 8) || (n && overlaps(sorted, n * 8, out, q * 8)))
    return fail(FS_ERR_INVALID_ARGUMENT, "out overlaps an input");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_bound_u64(sorted, n, queries, q, upper, out, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_bound_u64");
  return finish(s, "fs_bound_u64");
}

// ------------------------------------------------------------ NEXT-2: fused expand-to-peer
size_t fs_expand_to_peers_u16_temp_bytes(uint64_t nbins, int G) {
  return (nbins == 0 || nbins > 65536 || G < 1 || G > 1024) ? 0 : expand_to_peers_temp_bytes(nbins, G);
}

fs_status fs_expand_to_peers_u16(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint16_t* const* dest,
                                 void* temp, size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (G < 1 || G > 1024 || g < 0 || g >= G) return fail(FS_ERR_INVALID_ARGUMENT, "bad G=%d g=%d", G, g);
  if (nbins == 0 || nbins > 65536) return fail(FS_ERR_INVALID_ARGUMENT, "nbins not in 1..65536");
  if (!hist_all || !dest || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  for (int d = 0; d < G; ++d)
    if (!dest[d]) return fail(FS_ERR_INVALID_ARGUMENT, "dest[%d] is NULL", d);
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "temp not 256-byte aligned");
  const size_t need = expand_to_peers_temp_bytes(nbins, G);
  if (temp_bytes < need) return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_expand_to_peers(hist_all, G, g, nbins, dest, temp, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_expand_to_peers_u16");
  return finish(s, "fs_expand_to_peers_u16");
}

// ------------------------------------------------------------ NEXT-3: order statistics
size_t fs_trie_levels_count(int p) { return (p < 1 || p > 24) ? 0 : (((size_t)2 << p) - 1); }

fs_status fs_trie_levels(const uint64_t* leaf_hist, int p, uint64_t* levels, fs_stream_t stream) {
  FS_ENTRY();
  if (p < 1 || p > 24) return fail(FS_ERR_INVALID_ARGUMENT, "p %d not in 1..24", p);
  if (!leaf_hist || !levels) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (overlaps(leaf_hist, ((size_t)1 << p) * 8, levels, fs_trie_levels_count(p) * 8))
    return fail(FS_ERR_INVALID_ARGUMENT, "leaf_hist and levels overlap");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_trie_levels(leaf_hist, p, levels, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_trie_levels");
  return finish(s, "fs_trie_levels");
}

static int bitlen_u64(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

size_t fs_trie_pack_words(int p, uint64_t capacity) {
  if (p < 1 || p > 24) return 0;
  // widths never exceed bitlen(capacity) + 3 when every count <= capacity
  int full = bitlen_u64(capacity);
  uint64_t bits = 0;
  for (int l = 0; l <= p; ++l) {
    int w = full + 3;
    if (w > 64) w = 64;
    bits += ((uint64_t)1 << l) * (uint64_t)w;
  }
  return (size_t)((bits + 63) / 64);
}

size_t fs_trie_pack_temp_bytes(int p) { return (p < 1 || p > 24) ? 0 : align_up(sizeof(uint64_t) * (p + 1)); }

fs_status fs_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int32_t* widths,
                       uint64_t* bit_offsets, uint64_t* packed, uint64_t packed_words, void* temp,
                       size_t temp_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (p < 1 || p > 24) return fail(FS_ERR_INVALID_ARGUMENT, "p %d not in 1..24", p);
  if (min_width < 1 || min_width > 64) return fail(FS_ERR_INVALID_ARGUMENT, "min_width %d not in 1..64", min_width);
  if (!levels || !widths || !bit_offsets || !packed || !temp) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (temp_bytes < fs_trie_pack_temp_bytes(p))
    return fail(FS_ERR_INVALID_ARGUMENT, "temp_bytes %zu < required %zu", temp_bytes, fs_trie_pack_temp_bytes(p));
  if (packed_words == 0) return fail(FS_ERR_INVALID_ARGUMENT, "packed_words is 0");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_trie_pack(levels, p, capacity, min_width, widths, bit_offsets, packed, packed_words,
                                   (unsigned long long*)temp, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_trie_pack");
  return finish(s, "fs_trie_pack");
}

fs_status fs_get_item(const int32_t* widths, const uint64_t* bit_offsets, const uint64_t* packed, int p,
                      const uint64_t* ranks, uint64_t q, uint64_t default_value, uint64_t* items,
                      fs_stream_t stream) {
  FS_ENTRY();
  if (p < 1 || p > 24) return fail(FS_ERR_INVALID_ARGUMENT, "p %d not in 1..24", p);
  if (q == 0) return FS_OK;
  if (!widths || !bit_offsets || !packed || !ranks || !items) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_get_item(widths, bit_offsets, packed, p, ranks, q, default_value, items, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_get_item");
  return finish(s, "fs_get_item");
}

fs_status fs_get_index(const int32_t* widths, const uint64_t* bit_offsets, const uint64_t* packed, int p,
                       const uint64_t* values, uint64_t q, uint64_t* indices, fs_stream_t stream) {
  FS_ENTRY();
  if (p < 1 || p > 24) return fail(FS_ERR_INVALID_ARGUMENT, "p %d not in 1..24", p);
  if (q == 0) return FS_OK;
  if (!widths || !bit_offsets || !packed || !values || !indices)
    return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_get_index(widths, bit_offsets, packed, p, values, q, indices, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_get_index");
  return finish(s, "fs_get_index");
}

fs_status fs_hist_merge_u64(const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t count,
                            fs_stream_t stream) {
  FS_ENTRY();
  if (count == 0) return FS_OK;
  if (!a || !b || !out) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_hist_merge(a, b, out, count, s);
  if (e != cudaSuccess) return cuda_fail(e, "fs_hist_merge_u64");
  return finish(s, "fs_hist_merge_u64");
}

static fs_status wide_sort(const char* name, const void* kin, const uint32_t* vin, void* kout, uint32_t* vout,
                           uint64_t n, int key_bytes, int key_bits, void* temp, size_t temp_bytes,
                           fs_stream_t stream) {
  FS_ENTRY();
  const int width = key_bytes * 8;
  if (key_bits < 0 || key_bits > width) return fail(FS_ERR_INVALID_ARGUMENT, "%s: key_bits %d not in 0..%d", name,
                                                    key_bits, width);
  if (key_bits == 0) key_bits = width;
  if (n == 0) return FS_OK;
  const bool pairs = vout != nullptr || vin != nullptr;
  if (!kin || !kout || !temp || (pairs && (!vin || !vout)))
    return fail(FS_ERR_INVALID_ARGUMENT, "%s: NULL pointer with n > 0", name);
  if ((uintptr_t)temp & 255) return fail(FS_ERR_INVALID_ARGUMENT, "%s: temp not 256-byte aligned", name);
  if (((uintptr_t)kin | (uintptr_t)kout) & (key_bytes - 1))
    return fail(FS_ERR_INVALID_ARGUMENT, "%s: keys misaligned", name);
  if (pairs && (((uintptr_t)vin | (uintptr_t)vout) & 3))
    return fail(FS_ERR_INVALID_ARGUMENT, "%s: values misaligned", name);
  const size_t need = wide_temp_bytes(n, key_bytes, key_bits, pairs);
  if (temp_bytes < need) return fail(FS_ERR_INVALID_ARGUMENT, "%s: temp_bytes %zu < required %zu", name, temp_bytes,
                                     need);
  const size_t kb = (size_t)n * key_bytes, vb = (size_t)n * 4;
  if (overlaps(kin, kb, kout, kb) || (pairs && (overlaps(vin, vb, vout, vb) || overlaps(kin, kb, vout, vb) ||
                                                overlaps(vin, vb, kout, kb) || overlaps(kout, kb, vout, vb))))
    return fail(FS_ERR_INVALID_ARGUMENT, "%s: input and output buffers overlap", name);
  if (overlaps(temp, need, kin, kb) || overlaps(temp, need, kout, kb) ||
      (pairs && (overlaps(temp, need, vin, vb) || overlaps(temp, need, vout, vb))))
    return fail(FS_ERR_INVALID_ARGUMENT, "%s: temp overlaps a data buffer", name);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = wide_sort(kin, vin, kout, vout, n, key_bytes, key_bits, temp, temp_bytes, s);
  if (e != cudaSuccess) return cuda_fail(e, name);
  return finish(s, name);
}

fs_status fs_sort_keys_u32(const uint32_t* keys_in, uint32_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream) {
  return wide_sort("fs_sort_keys_u32", keys_in, nullptr, keys_out, nullptr, n, 4, key_bits, temp, temp_bytes,
                   stream);
}

fs_status fs_sort_keys_u64(const uint64_t* keys_in, uint64_t* keys_out, uint64_t n, int key_bits, void* temp,
                           size_t temp_bytes, fs_stream_t stream) {
  return wide_sort("fs_sort_keys_u64", keys_in, nullptr, keys_out, nullptr, n, 8, key_bits, temp, temp_bytes,
                   stream);
}

fs_status fs_sort_pairs_u64_u32(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                                uint32_t* vals_out, uint64_t n, int key_bits, void* temp, size_t temp_bytes,
                                fs_stream_t stream) {
  if (n && (!vals_in || !vals_out)) {
    FS_ENTRY();
    return fail(FS_ERR_INVALID_ARGUMENT, "fs_sort_pairs_u64_u32: NULL values with n > 0");
  }
  return wide_sort("fs_sort_pairs_u64_u32", keys_in, vals_in, keys_out, vals_out, n, 8, key_bits, temp,
                   temp_bytes, stream);
}

}  // extern "C"
