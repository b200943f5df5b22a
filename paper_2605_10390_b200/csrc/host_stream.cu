// host_stream.cu — fs_sort_keys_u16_host: the u16 sort from host memory to host
// memory, streamed in batches (the runtime around the kernels; G11 / NEXT-4).
//
// Batch Size Selection and Batch Counter Update (§III.C-D):
// the input streams in input order in equal batches; the histogram of every
// batch is added into one reused histogram (fs_histogram_u16 accumulate = 1), so
// batch switching costs no histogram rebuild.  After the last batch the scan
// runs once and the output is reconstructed batch by batch (fs_expand_u16 over
// output ranges) and streamed back.  Copies run on two private copy streams --
// host->device on one, device->host on the other, so the two directions of the
// PCIe link (two copy engines) can overlap -- and overlap the kernels of the
// neighbouring batch (double-buffered device slots).  Within one call the
// output cannot start before the last input batch is counted; calls issued on
// different streams with their own work buffers overlap one call's output with
// the next call's input.
#include <cuda_runtime.h>

#include "fractalsort.h"
#include "internal.cuh"
#include "kernels.cuh"

namespace fs {
namespace {

constexpr uint64_t kDefaultBatch = 1ull << 24;  // 32 MB of keys per copy

struct HostLayout {
  uint64_t batch = 0;
  size_t buf0 = 0, buf1 = 0, hist = 0, prefix = 0, htemp = 0, htemp_bytes = 0, stemp = 0, stemp_bytes = 0,
         total = 0;
};

HostLayout host_layout(uint64_t n, uint64_t batch) {
  HostLayout L;
  if (batch == 0) batch = kDefaultBatch;
  batch = (batch + 7) / 8 * 8;  // keep every slot 16-byte aligned
  if (batch > n) batch = (n + 7) / 8 * 8;
  if (batch == 0) batch = 8;
  L.batch = batch;
  size_t off = 0;
  L.buf0 = off;
  off = align_up(off + batch * 2);
  L.buf1 = off;
  off = align_up(off + batch * 2);
  L.hist = off;
  off = align_up(off + 8 * kHistBins);
  L.prefix = off;
  off = align_up(off + 8 * (kHistBins + 1));
  L.htemp = off;
  L.htemp_bytes = fs_histogram_u16_temp_bytes(batch);
  off = align_up(off + L.htemp_bytes);
  L.stemp = off;
  L.stemp_bytes = fs_exclusive_scan_u64_temp_bytes(kHistBins);
  off = align_up(off + L.stemp_bytes);
  L.total = off;
  return L;
}

// The copy streams (in: H2D, out: D2H) and 9 events, created on first use and
// kept for the life of the process: one set per host thread and device (a thread's calls are
// issued in order, so re-recording an event in a later call is safe -- a wait
// captures the record current at the time of the wait; calls from other threads
// use their own set).  No per-call stream or event creation.
constexpr int kMaxDevices = 64;
struct Resources {
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev[9] = {};
  bool ready = false;
};
thread_local Resources t_res[kMaxDevices];

cudaError_t resources(Resources*& R) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  R = &t_res[dev];
  if (R->ready) return cudaSuccess;
  if (!R->copy_in && (e = cudaStreamCreateWithFlags(&R->copy_in, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if (!R->copy_out && (e = cudaStreamCreateWithFlags(&R->copy_out, cudaStreamNonBlocking)) != cudaSuccess) return e;
  for (int i = 0; i < 9; ++i)
    if (!R->ev[i] && (e = cudaEventCreateWithFlags(&R->ev[i], cudaEventDisableTiming)) != cudaSuccess) return e;
  R->ready = true;
  return cudaSuccess;
}

}  // namespace
}  // namespace fs

using namespace fs;

extern "C" {

size_t fs_sort_keys_u16_host_work_bytes(uint64_t n, uint64_t batch) { return host_layout(n, batch).total; }

fs_status fs_sort_keys_u16_host(const uint16_t* keys_in_host, uint16_t* keys_out_host, uint64_t n, uint64_t batch,
                                void* work, size_t work_bytes, fs_stream_t stream) {
  FS_ENTRY();
  if (n == 0) return FS_OK;
  if (!keys_in_host || !keys_out_host || !work) return fail(FS_ERR_INVALID_ARGUMENT, "NULL pointer with n > 0");
  if ((uintptr_t)work & 255) return fail(FS_ERR_INVALID_ARGUMENT, "work not 256-byte aligned");
  const HostLayout L = host_layout(n, batch);
  if (work_bytes < L.total) return fail(FS_ERR_INVALID_ARGUMENT, "work_bytes %zu < required %zu", work_bytes, L.total);
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)work;
  uint16_t* buf[2] = {(uint16_t*)(w + L.buf0), (uint16_t*)(w + L.buf1)};
  uint64_t* hist = (uint64_t*)(w + L.hist);
  uint64_t* prefix = (uint64_t*)(w + L.prefix);

  Resources* R = nullptr;
  cudaError_t e = resources(R);
  if (e != cudaSuccess) return cuda_fail(e, "fs_sort_keys_u16_host: copy stream/event create");
  cudaEvent_t* copied = R->ev;       // [2]
  cudaEvent_t* consumed = R->ev + 2; // [2] slot free again (hist or D2H done)
  cudaEvent_t* expanded = R->ev + 4; // [2]
  cudaEvent_t start = R->ev[6];
  cudaEvent_t done_in = R->ev[7];
  cudaEvent_t done_out = R->ev[8];
  // On an error after work was queued: order everything later on `stream` after
  // the copies already queued on both copy streams (nothing is left dangling).
  auto drain = [&](fs_status st) {
    if (cudaEventRecord(done_in, R->copy_in) == cudaSuccess) cudaStreamWaitEvent(s, done_in, 0);
    if (cudaEventRecord(done_out, R->copy_out) == cudaSuccess) cudaStreamWaitEvent(s, done_out, 0);
    return st;
  };

  // The input copies start after whatever the caller queued earlier on `stream`.
  cudaEventRecord(start, s);
  cudaStreamWaitEvent(R->copy_in, start, 0);

  const uint64_t B = L.batch, nb = (n + B - 1) / B;
  // ---- phase 1: stream batches in, one reused histogram
  for (uint64_t i = 0; i < nb; ++i) {
    const int slot = (int)(i & 1);
    const uint64_t len = (i + 1) * B <= n ? B : n - i * B;
    if (i >= 2) cudaStreamWaitEvent(R->copy_in, consumed[slot], 0);
    e = cudaMemcpyAsync(buf[slot], keys_in_host + i * B, len * 2, cudaMemcpyHostToDevice, R->copy_in);
    if (e != cudaSuccess) return drain(cuda_fail(e, "fs_sort_keys_u16_host: H2D"));
    cudaEventRecord(copied[slot], R->copy_in);
    cudaStreamWaitEvent(s, copied[slot], 0);
    fs_status st = fs_histogram_u16(buf[slot], len, 16, hist, i > 0, w + L.htemp, L.htemp_bytes, stream);
    if (st != FS_OK) return drain(st);
    cudaEventRecord(consumed[slot], s);
  }
  // ---- phase 2: one scan of the merged histogram
  fs_status st = fs_exclusive_scan_u64(hist, prefix, kHistBins, w + L.stemp, L.stemp_bytes, stream);
  if (st != FS_OK) return drain(st);
  // ---- phase 3: reconstruct batch by batch and stream out (slots 0 and 1 were
  //      last read by histograms on `stream`: stream order covers them)
  for (uint64_t j = 0; j < nb; ++j) {
    const int slot = (int)(j & 1);
    const uint64_t len = (j + 1) * B <= n ? B : n - j * B;
    if (j >= 2) cudaStreamWaitEvent(s, consumed[slot], 0);
    st = fs_expand_u16(prefix, kHistBins, j * B, j * B + len, buf[slot], stream);
    if (st != FS_OK) return drain(st);
    cudaEventRecord(expanded[slot], s);
    cudaStreamWaitEvent(R->copy_out, expanded[slot], 0);
    e = cudaMemcpyAsync(keys_out_host + j * B, buf[slot], len * 2, cudaMemcpyDeviceToHost, R->copy_out);
    if (e != cudaSuccess) return drain(cuda_fail(e, "fs_sort_keys_u16_host: D2H"));
    cudaEventRecord(consumed[slot], R->copy_out);
  }
  cudaEventRecord(done_out, R->copy_out);
  cudaStreamWaitEvent(s, done_out, 0);  // synchronising `stream` now implies the output is on the host
  return finish(s, "fs_sort_keys_u16_host");
}

}  // extern "C"
