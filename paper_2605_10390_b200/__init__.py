"""paper_2605_10390_b200 — B200-native compressed-histogram radix sort (FractalSortCPU,
arXiv 2605.10390), as a thin Python binding over libfractalsort.so.

Every step of the sort runs in the library's sm_100a kernels; this module only
marshals arguments: it allocates outputs and temp buffers with torch, passes raw
device pointers and the current CUDA stream to the C ABI (include/fractalsort.h)
and raises on a non-OK status.  There is no CPU fallback: CPU tensors raise.

Names follow the C ABI: sort_keys (fs_sort_keys_u16/u32/u64), sort_pairs
(fs_sort_pairs_u64_u32), histogram_u16 / exclusive_scan / expand_u16 (the phase
API), send_counts (multi-GPU exchange plan) and sort_keys_u16_host (host
buffers, streamed in batches).
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import FractalSortError, check, lib

__all__ = [
    "sort_keys", "sort_pairs", "histogram_u16", "exclusive_scan", "expand_u16", "send_counts",
    "sort_keys_u16_host", "sort_keys_u16_host_work_bytes", "FractalSortError", "lib",
    "histogram_prefix_u16", "expand_prefix_u16", "expand_to_peers_u16", "bound_u64", "trie_levels", "PackedTrie",
    "trie_pack", "get_item", "get_index", "hist_merge", "histogram16_u64", "select_bins_u64",
    "digit_counts_sorted_u64", "PairExchange", "allreduce_multicast_u64",
]

_TEMP_ALIGN = 256


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(*ts: torch.Tensor) -> torch.device:
    dev = ts[0].device
    for t in ts:
        if t.device.type != "cuda":
            raise ValueError("paper_2605_10390_b200 runs on CUDA tensors only (no CPU fallback)")
        if t.device != dev:
            raise ValueError("all tensors must be on the same device")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
    return dev


def _temp(nbytes: int, device: torch.device) -> torch.Tensor:
    # torch's caching allocator returns >= 512-byte aligned blocks.
    t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
    assert t.data_ptr() % _TEMP_ALIGN == 0
    return t


def sort_keys(keys: torch.Tensor, key_bits: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Ascending keys-only sort of a 1-D uint16/uint32/uint64 CUDA tensor.

    uint16 -> fs_sort_keys_u16 (histogram, scan, count-expansion — one 16-CTA cluster
    launch for n <= 2^18, else two kernels; out may be keys);
    uint32/uint64 -> fs_sort_keys_u32/u64 (trie-binned MSD with a per-bin shared-memory sort
    for n > 8,960 and key_bits >= 32 — oversize bins recurse on the next digits, the window
    moves below a common key prefix — else LSD with one compressed histogram per 8-bit digit;
    decided on the device).
    """
    dev = _require_cuda(keys)
    n = keys.numel()
    if out is None:
        out = torch.empty_like(keys)
    else:
        _require_cuda(out)
        if out.dtype != keys.dtype or out.numel() != n:
            raise ValueError("out must match keys in dtype and size")
    L = lib()
    with torch.cuda.device(dev):
        s = _stream(dev)
        if keys.dtype == torch.uint16:
            temp = _temp(L.fs_sort_keys_u16_temp_bytes(n), dev)
            check(L.fs_sort_keys_u16(keys.data_ptr(), out.data_ptr(), n, key_bits, temp.data_ptr(),
                                     temp.numel(), s), "fs_sort_keys_u16")
        elif keys.dtype == torch.uint32:
            temp = _temp(L.fs_sort_keys_u32_temp_bytes(n, key_bits), dev)
            check(L.fs_sort_keys_u32(keys.data_ptr(), out.data_ptr(), n, key_bits, temp.data_ptr(),
                                     temp.numel(), s), "fs_sort_keys_u32")
        elif keys.dtype == torch.uint64:
            temp = _temp(L.fs_sort_keys_u64_temp_bytes(n, key_bits), dev)
            check(L.fs_sort_keys_u64(keys.data_ptr(), out.data_ptr(), n, key_bits, temp.data_ptr(),
                                     temp.numel(), s), "fs_sort_keys_u64")
        else:
            raise TypeError(f"unsupported key dtype {keys.dtype}")
    return out


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, key_bits: int = 0):
    """Stable ascending sort of (uint64 key, uint32 value) pairs by key (fs_sort_pairs_u64_u32)."""
    dev = _require_cuda(keys, vals)
    if keys.dtype != torch.uint64 or vals.dtype != torch.uint32 or keys.numel() != vals.numel():
        raise TypeError("sort_pairs expects uint64 keys and uint32 values of equal length")
    n = keys.numel()
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_sort_pairs_u64_u32_temp_bytes(n, key_bits), dev)
        check(L.fs_sort_pairs_u64_u32(keys.data_ptr(), vals.data_ptr(), ko.data_ptr(), vo.data_ptr(), n,
                                      key_bits, temp.data_ptr(), temp.numel(), _stream(dev)),
              "fs_sort_pairs_u64_u32")
    return ko, vo


def histogram_u16(keys: torch.Tensor, key_bits: int = 16, hist: torch.Tensor | None = None,
                  accumulate: bool = False) -> torch.Tensor:
    """hist[v] (+)= #{i: keys[i] == v} (fs_histogram_u16); hist is int64 (bit-identical to u64)."""
    dev = _require_cuda(keys)
    if keys.dtype != torch.uint16:
        raise TypeError("histogram_u16 expects uint16 keys")
    nb = 1 << (key_bits or 16)
    if hist is None:
        hist = torch.empty(nb, dtype=torch.int64, device=dev)
        accumulate = False
    elif hist.numel() != nb or hist.dtype not in (torch.int64, torch.uint64):
        raise ValueError("hist must hold 2^key_bits int64/uint64 counters")
    n = keys.numel()
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_histogram_u16_temp_bytes(n), dev)
        check(L.fs_histogram_u16(keys.data_ptr(), n, key_bits, hist.data_ptr(), int(bool(accumulate)),
                                 temp.data_ptr(), temp.numel(), _stream(dev)), "fs_histogram_u16")
    return hist


def histogram_prefix_u16(keys: torch.Tensor, prefix2: torch.Tensor | None = None, out_ptr: int | None = None):
    """The sort's two-level prefix of keys: 65,536 slice-local prefixes + 128 slice totals, int64
    (fs_histogram_prefix_u16); sums over ranks stay in the same form.  ``out_ptr``: write them
    to this raw device address instead (e.g. a multicast-bound buffer, dist.MulticastBuffer)
    and return None."""
    dev = _require_cuda(keys)
    if keys.dtype != torch.uint16:
        raise TypeError("histogram_prefix_u16 expects uint16 keys")
    if out_ptr is None and prefix2 is None:
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
    n = keys.numel()
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_histogram_u16_temp_bytes(n), dev)
        check(L.fs_histogram_prefix_u16(keys.data_ptr(), n, out_ptr if out_ptr is not None else prefix2.data_ptr(),
                                        temp.data_ptr(), temp.numel(), _stream(dev)), "fs_histogram_prefix_u16")
    return None if out_ptr is not None else prefix2


def allreduce_multicast_u64(src_mc: int, dst: torch.Tensor, flag_mc: int, flag_local: int, target: int,
                            timed_out: torch.Tensor | None = None, timeout_s: float = 60.0):
    """dst[i] = sum over ranks of their src[i] (int64/uint64 dst, i < dst.numel()), read through the
    multicast address src_mc by multimem.ld_reduce, with the call's cross-GPU barrier on the
    flag word (fs_allreduce_multicast_u64; addresses from dist.MulticastBuffer).  ``timed_out``:
    a device int32[1], zeroed here, set to 1 by the kernel if the peers did not all arrive within
    ``timeout_s`` (dst is then not written); check it after synchronising.  Returns (dst, timed_out)."""
    dev = _require_cuda(dst)
    if dst.dtype not in (torch.int64, torch.uint64) or not dst.is_contiguous():
        raise TypeError("dst must be a contiguous 64-bit integer tensor")
    if timed_out is None:
        timed_out = torch.zeros(1, dtype=torch.int32, device=dev)
    else:
        timed_out.zero_()
    with torch.cuda.device(dev):
        check(lib().fs_allreduce_multicast_u64(src_mc, dst.data_ptr(), dst.numel(), flag_mc, flag_local,
                                               target & 0xFFFFFFFF, int(timeout_s * 1e9), timed_out.data_ptr(),
                                               _stream(dev)), "fs_allreduce_multicast_u64")
    return dst, timed_out


def expand_prefix_u16(prefix2: torch.Tensor, out_begin: int, out_end: int, out: torch.Tensor | None = None):
    """Keys at global sorted positions [out_begin, out_end) from a two-level prefix (fs_expand_prefix_u16)."""
    dev = _require_cuda(prefix2)
    n = out_end - out_begin
    if out is None:
        out = torch.empty(n, dtype=torch.uint16, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_expand_prefix_u16(prefix2.data_ptr(), out_begin, out_end, out.data_ptr(), _stream(dev)),
              "fs_expand_prefix_u16")
    return out


def exclusive_scan(hist: torch.Tensor) -> torch.Tensor:
    """prefix[v] = sum_{u<v} hist[u], prefix[nbins] = total (fs_exclusive_scan_u64)."""
    dev = _require_cuda(hist)
    if hist.dtype not in (torch.int64, torch.uint64):
        raise TypeError("exclusive_scan expects int64/uint64 counts")
    nb = hist.numel()
    prefix = torch.empty(nb + 1, dtype=hist.dtype, device=dev)
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_exclusive_scan_u64_temp_bytes(nb), dev)
        check(L.fs_exclusive_scan_u64(hist.data_ptr(), prefix.data_ptr(), nb, temp.data_ptr(), temp.numel(),
                                      _stream(dev)), "fs_exclusive_scan_u64")
    return prefix


def expand_u16(prefix: torch.Tensor, out_begin: int, out_end: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Keys at global sorted positions [out_begin, out_end) from a prefix array (fs_expand_u16)."""
    dev = _require_cuda(prefix)
    n = out_end - out_begin
    if out is None:
        out = torch.empty(n, dtype=torch.uint16, device=dev)
    elif out.dtype != torch.uint16 or out.numel() < n:
        raise ValueError("out must be uint16 with room for out_end - out_begin keys")
    with torch.cuda.device(dev):
        check(lib().fs_expand_u16(prefix.data_ptr(), prefix.numel() - 1, out_begin, out_end, out.data_ptr(),
                                  _stream(dev)), "fs_expand_u16")
    return out


def send_counts(hist_all: torch.Tensor, g: int) -> torch.Tensor:
    """send[d] = how many of rank g's keys land in rank d's output range (fs_send_counts)."""
    dev = _require_cuda(hist_all)
    G, nb = hist_all.shape
    send = torch.empty(G, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_send_counts(hist_all.data_ptr(), G, g, nb, send.data_ptr(), _stream(dev)),
              "fs_send_counts")
    return send


def bound_u64(sorted_keys: torch.Tensor, queries: torch.Tensor, upper: bool = False) -> torch.Tensor:
    """#keys < q (upper=False) or <= q (upper=True) in an ascending uint64 tensor (fs_bound_u64)."""
    dev = _require_cuda(sorted_keys, queries)
    out = torch.empty(queries.numel(), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_bound_u64(sorted_keys.data_ptr(), sorted_keys.numel(), queries.data_ptr(), queries.numel(),
                                 int(bool(upper)), out.data_ptr(), _stream(dev)), "fs_bound_u64")
    return out


def histogram16_u64(keys: torch.Tensor, shift: int, width: int = 16) -> torch.Tensor:
    """int64[2^width]: histogram of the digit (keys >> shift) & (2^width - 1) (fs_histogram16_u64)."""
    dev = _require_cuda(keys)
    if keys.dtype != torch.uint64:
        raise TypeError("histogram16_u64 expects uint64 keys")
    hist = torch.empty(1 << width, dtype=torch.int64, device=dev)
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_histogram16_u64_temp_bytes(keys.numel()), dev)
        check(L.fs_histogram16_u64(keys.data_ptr(), keys.numel(), shift, width, hist.data_ptr(), temp.data_ptr(),
                                   temp.numel(), _stream(dev)), "fs_histogram16_u64")
    return hist


def select_bins_u64(keys: torch.Tensor, shift: int, width: int, bins: list, cap: int) -> torch.Tensor:
    """The keys whose digit (keys >> shift) & (2^width - 1) is one of `bins`, in no
    particular order (fs_select_bins_u64); cap must be at least their number."""
    dev = _require_cuda(keys)
    b = torch.tensor(list(bins), dtype=torch.int32, device=dev)
    out = torch.empty(max(int(cap), 1), dtype=torch.uint64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_select_bins_u64(keys.data_ptr(), keys.numel(), shift, width, b.data_ptr(), b.numel(),
                                       out.data_ptr(), int(cap), count.data_ptr(), _stream(dev)), "fs_select_bins_u64")
    m = int(count.item())
    if m > cap:
        raise ValueError(f"select_bins_u64: {m} keys match, cap {cap}")
    return out[:m]


def digit_counts_sorted_u64(sorted_keys: torch.Tensor, prefixes: list, shift: int, width: int = 16) -> torch.Tensor:
    """int64[len(prefixes), 2^width]: per prefix, the histogram of the digit at
    `shift` among the keys sharing the prefix's bits above it (fs_digit_counts_sorted_u64)."""
    dev = _require_cuda(sorted_keys)
    np_ = len(prefixes)
    hist = torch.empty((np_, 1 << width), dtype=torch.int64, device=dev)
    if np_ == 0:
        return hist
    import numpy as np
    p = torch.from_numpy(np.array(prefixes, dtype=np.uint64).view(np.int64)).to(dev)
    with torch.cuda.device(dev):
        check(lib().fs_digit_counts_sorted_u64(sorted_keys.data_ptr(), sorted_keys.numel(), p.data_ptr(), np_,
                                               shift, width, hist.data_ptr(), _stream(dev)),
              "fs_digit_counts_sorted_u64")
    return hist


class PairExchange:
    """The fused partition-to-peer exchange of the distributed pair sort
    (fs_pair_classes_u64, then fs_pair_scatter_u64_u32 with the same temp)."""

    def __init__(self, keys: torch.Tensor, vals: torch.Tensor, splitters: list, G: int):
        import numpy as np
        self.dev = _require_cuda(keys, vals)
        self.keys, self.vals, self.G = keys, vals, G
        self.K = torch.from_numpy(np.array(splitters if splitters else [0], dtype=np.uint64).view(np.int64)).to(self.dev)
        L = lib()
        self.temp = _temp(L.fs_pair_exchange_temp_bytes(keys.numel(), G), self.dev)

    def classes(self) -> list:
        """Class totals (2G - 1 counts: class 2d = strictly inside owner d's key range, 2d + 1 = equal to K_d)."""
        tot = torch.empty(2 * self.G - 1, dtype=torch.int64, device=self.dev)
        with torch.cuda.device(self.dev):
            check(lib().fs_pair_classes_u64(self.keys.data_ptr(), self.keys.numel(), self.K.data_ptr(), self.G,
                                            tot.data_ptr(), self.temp.data_ptr(), self.temp.numel(),
                                            _stream(self.dev)), "fs_pair_classes_u64")
        return [int(x) for x in tot.tolist()]

    def scatter(self, cuts: list, bases: list, dest_keys: list, dest_vals: list) -> None:
        import ctypes
        G = self.G
        c = (ctypes.c_uint64 * (G + 1))(*[int(x) for x in cuts])
        b = (ctypes.c_uint64 * G)(*[int(x) for x in bases])
        dk = (ctypes.c_void_p * G)(*[t.data_ptr() for t in dest_keys])
        dv = (ctypes.c_void_p * G)(*[t.data_ptr() for t in dest_vals])
        with torch.cuda.device(self.dev):
            check(lib().fs_pair_scatter_u64_u32(self.keys.data_ptr(), self.vals.data_ptr(), self.keys.numel(),
                                                self.K.data_ptr(), G, c, b, dk, dv, self.temp.data_ptr(),
                                                self.temp.numel(), _stream(self.dev)), "fs_pair_scatter_u64_u32")


def expand_to_peers_u16(hist_all: torch.Tensor, g: int, dest: list) -> None:
    """Rank g writes its keys to their final sorted positions in dest[d] (the
    buffer of the rank owning them; peer-mapped tensors), fs_expand_to_peers_u16."""
    import ctypes
    dev = _require_cuda(hist_all)
    G, nb = hist_all.shape
    if len(dest) != G:
        raise ValueError("dest must hold one buffer per rank")
    ptrs = (ctypes.c_void_p * G)(*[t.data_ptr() for t in dest])
    L = lib()
    with torch.cuda.device(dev):
        temp = _temp(L.fs_expand_to_peers_u16_temp_bytes(nb, G), dev)
        check(L.fs_expand_to_peers_u16(hist_all.data_ptr(), G, g, nb, ptrs, temp.data_ptr(), temp.numel(),
                                       _stream(dev)), "fs_expand_to_peers_u16")


def sort_keys_u16_host_work_bytes(n: int, batch: int = 0) -> int:
    return int(lib().fs_sort_keys_u16_host_work_bytes(n, batch))


def sort_keys_u16_host(keys_host: torch.Tensor, out_host: torch.Tensor | None = None, batch: int = 0,
                       device: torch.device | int | None = None, work: torch.Tensor | None = None,
                       synchronize: bool = True) -> torch.Tensor:
    """Sort host-resident uint16 keys into a host tensor through the device (fs_sort_keys_u16_host).

    Pass pinned tensors (``tensor.pin_memory()``) for overlapped copies.
    """
    if keys_host.device.type != "cpu" or keys_host.dtype != torch.uint16 or not keys_host.is_contiguous():
        raise ValueError("keys_host must be a contiguous uint16 CPU tensor")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       (device if isinstance(device, int) else device.index or 0))
    n = keys_host.numel()
    if out_host is None:
        out_host = torch.empty(n, dtype=torch.uint16, pin_memory=keys_host.is_pinned())
    L = lib()
    with torch.cuda.device(dev):
        need = L.fs_sort_keys_u16_host_work_bytes(n, batch)
        if work is None or work.numel() < need:
            work = _temp(need, dev)
        s = _stream(dev)
        check(L.fs_sort_keys_u16_host(keys_host.data_ptr(), out_host.data_ptr(), n, batch, work.data_ptr(),
                                      work.numel(), s), "fs_sort_keys_u16_host")
        if synchronize:
            torch.cuda.current_stream(dev).synchronize()
    return out_host


# ---------------------------------------------------------------- order statistics (NEXT-3)
def trie_levels(leaf_hist: torch.Tensor, p: int) -> torch.Tensor:
    """Dense trie levels (2^(p+1) - 1 int64, level l at offset 2^l - 1) from a 2^p leaf histogram."""
    dev = _require_cuda(leaf_hist)
    if leaf_hist.dtype not in (torch.int64, torch.uint64) or leaf_hist.numel() != (1 << p):
        raise ValueError("leaf_hist must hold 2^p int64/uint64 counters")
    L = lib()
    levels = torch.empty(L.fs_trie_levels_count(p), dtype=leaf_hist.dtype, device=dev)
    with torch.cuda.device(dev):
        check(L.fs_trie_levels(leaf_hist.data_ptr(), p, levels.data_ptr(), _stream(dev)), "fs_trie_levels")
    return levels


class PackedTrie:
    """A tapered bit-packed trie on the device (fs_trie_pack output)."""

    def __init__(self, p: int, widths: torch.Tensor, bit_offsets: torch.Tensor, packed: torch.Tensor):
        self.p, self.widths, self.bit_offsets, self.packed = p, widths, bit_offsets, packed


def trie_pack(levels: torch.Tensor, p: int, capacity: int, min_width: int = 1) -> PackedTrie:
    dev = _require_cuda(levels)
    L = lib()
    words = L.fs_trie_pack_words(p, capacity)
    widths = torch.empty(p + 1, dtype=torch.int32, device=dev)
    offs = torch.empty(p + 2, dtype=torch.int64, device=dev)
    packed = torch.empty(words, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        temp = _temp(L.fs_trie_pack_temp_bytes(p), dev)
        check(L.fs_trie_pack(levels.data_ptr(), p, capacity, min_width, widths.data_ptr(), offs.data_ptr(),
                             packed.data_ptr(), words, temp.data_ptr(), temp.numel(), _stream(dev)), "fs_trie_pack")
    return PackedTrie(p, widths, offs, packed)


def get_item(t: PackedTrie, ranks: torch.Tensor, default: int = 0) -> torch.Tensor:
    """Keys at ascending sorted ranks (Alg. 2), default where rank >= total (fs_get_item)."""
    dev = _require_cuda(ranks, t.packed)
    items = torch.empty(ranks.numel(), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_get_item(t.widths.data_ptr(), t.bit_offsets.data_ptr(), t.packed.data_ptr(), t.p,
                                ranks.data_ptr(), ranks.numel(), default, items.data_ptr(), _stream(dev)),
              "fs_get_item")
    return items


def get_index(t: PackedTrie, values: torch.Tensor) -> torch.Tensor:
    """#keys < value for each value (Alg. 3, fs_get_index)."""
    dev = _require_cuda(values, t.packed)
    idx = torch.empty(values.numel(), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        check(lib().fs_get_index(t.widths.data_ptr(), t.bit_offsets.data_ptr(), t.packed.data_ptr(), t.p,
                                 values.data_ptr(), values.numel(), idx.data_ptr(), _stream(dev)), "fs_get_index")
    return idx


def hist_merge(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = a + b, counter by counter (fs_hist_merge_u64)."""
    dev = _require_cuda(a, b)
    if a.numel() != b.numel():
        raise ValueError("a and b must have the same number of counters")
    out = torch.empty_like(a) if out is None else out
    with torch.cuda.device(dev):
        check(lib().fs_hist_merge_u64(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(), _stream(dev)),
              "fs_hist_merge_u64")
    return out
