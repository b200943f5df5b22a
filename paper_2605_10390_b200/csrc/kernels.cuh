// kernels.cuh — internal launch interface between the C ABI (abi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fs {

struct DeviceInfo {
  int device = 0;
  int sm_count = 0;
  int max_smem_optin = 0;
  int l2_bytes = 0;
  int cc_major = 0, cc_minor = 0;
};
// Cached per device, initialised thread-safely on first use (abi.cu).
const DeviceInfo& device_info();

// ---------------------------------------------------------------- hist16.cu
// Per-SM compressed histogram of u16 keys (stage 1).  One CTA per SM.
constexpr int kHistBins = 65536;
constexpr int kHistWords = kHistBins / 2;  // two 16-bit counters per 32-bit word
constexpr int kHistSlices = 128;            // 512-bin merge/scan slices
constexpr int kHistSpillWords = kHistBins + 32;  // spill[65536] + work counter (zeroed by the kernel)
int hist16_grid(uint64_t n);  // min(#SM, ceil(n / 65536))
// Cooperative launch, one CTA per SM: local histograms -> partials, grid sync,
// merge (C written to hist_out if non-null, += when accumulate), and, when
// prefix != nullptr, the two-level prefix: prefix[v] = sum of C over the bins of
// v's 512-bin slice below v, slice_tot[s] = total of slice s (kHistSlices).
// spill (65536 u64) is scratch; the kernel zeroes it itself.
cudaError_t launch_hist16(const uint16_t* keys, uint64_t n, uint32_t* partials, unsigned long long* spill,
                          uint64_t* hist_out, uint64_t nbins_out, int accumulate, uint64_t* prefix,
                          uint64_t* slice_tot, int grid, cudaStream_t s);

// ---------------------------------------------------------------- small16.cu
// The whole u16 keys-only sort in one launch of a 16-CTA cluster for n <=
// small16_max_n() (histogram in shared memory, merge of the 16 tables through
// L2, scan, expansion).  spill: 65,536 u64 of scratch (zeroed by the kernel);
// partials: 16 x kHistWords u32 of scratch.
uint64_t small16_max_n();
cudaError_t launch_sort16_small(const uint16_t* keys, uint64_t n, uint16_t* out, unsigned long long* spill,
                                uint32_t* partials, cudaStream_t s);

// ---------------------------------------------------------------- scan.cu
constexpr int kScanTileBins = 256;
inline uint64_t scan_tiles(uint64_t nbins) { return (nbins + kScanTileBins - 1) / kScanTileBins; }
// Merge + scan (stages 1b+2).  Source is either the packed per-SM partials plus
// spill (hist_in == nullptr) or a u64 histogram.  hist_out: nullptr, or written
// (accumulate = 0) / added to (accumulate = 1) for v < nbins_out.  prefix:
// nullptr (merge only) or nbins + 1 entries.  status (scan_tiles(nbins) u64)
// and *ticket must be zero on entry when prefix != nullptr.
cudaError_t launch_merge_scan(const uint32_t* partials, int parts, const unsigned long long* spill,
                              const uint64_t* hist_in, uint64_t nbins, uint64_t* hist_out, uint64_t nbins_out,
                              int accumulate, uint64_t* prefix, unsigned long long* status, uint32_t* ticket,
                              cudaStream_t s);

// ---------------------------------------------------------------- expand16.cu
// Count-expansion of prefix into out for global positions [out_begin, out_end) (stage 3).
cudaError_t launch_expand16(const uint64_t* prefix, uint64_t nbins, uint64_t out_begin, uint64_t out_end,
                            uint16_t* out, cudaStream_t s);
// Same from the two-level prefix written by launch_hist16 (65,536 bins).
cudaError_t launch_expand16_two_level(const uint64_t* slice_prefix, const uint64_t* slice_tot, uint64_t out_begin,
                                      uint64_t out_end, uint16_t* out, cudaStream_t s);

// ---------------------------------------------------------------- partition.cu
cudaError_t launch_send_counts(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint64_t* send,
                               cudaStream_t s);

cudaError_t launch_bound_u64(const uint64_t* sorted, uint64_t n, const uint64_t* q, uint64_t nq, int upper,
                             uint64_t* out, cudaStream_t s);

// ---------------------------------------------------------------- peer.cu
size_t expand_to_peers_temp_bytes(uint64_t nbins, int G);
cudaError_t launch_expand_to_peers(const uint64_t* hist_all, int G, int g, uint64_t nbins, uint16_t* const* dest_host,
                                   void* temp, cudaStream_t s);

// ---------------------------------------------------------------- trie.cu
// Order-statistic service (NEXT-3): dense levels, tapered bit-packed export, queries.
cudaError_t launch_trie_levels(const uint64_t* leaves, int p, uint64_t* levels, cudaStream_t s);
cudaError_t launch_trie_pack(const uint64_t* levels, int p, uint64_t capacity, int min_width, int32_t* widths,
                             uint64_t* off, uint64_t* packed, uint64_t words, unsigned long long* mx,
                             cudaStream_t s);
cudaError_t launch_get_item(const int32_t* widths, const uint64_t* off, const uint64_t* packed, int p,
                            const uint64_t* ranks, uint64_t q, uint64_t default_value, uint64_t* items,
                            cudaStream_t s);
cudaError_t launch_get_index(const int32_t* widths, const uint64_t* off, const uint64_t* packed, int p,
                             const uint64_t* values, uint64_t q, uint64_t* indices, cudaStream_t s);
cudaError_t launch_hist_merge(const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t count, cudaStream_t s);

// ---------------------------------------------------------------- wide.cu
// Stable sort of u32/u64 keys (+ optional u32 values): trie-binned MSD with a
// per-bin local sort when every 16-bit bin fits shared memory (decided on the
// device), else LSD radix with 8-bit digits.
size_t wide_temp_bytes(uint64_t n, int key_bytes, int key_bits, bool has_values);
bool wide_uses_msd(uint64_t n, int key_bytes, int key_bits);
cudaError_t wide_sort(const void* keys_in, const uint32_t* vals_in, void* keys_out, uint32_t* vals_out, uint64_t n,
                      int key_bytes, int key_bits, void* temp, size_t temp_bytes, cudaStream_t s);

}  // namespace fs
