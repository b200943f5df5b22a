"""ctypes wrapper of the plain CPU oracle (oracle/oracle.c -> liboracle.so).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product path (paper_2605_10390_b200/) never imports it and shares no code
with it.  Each wrapped function cites its paper passage in oracle/oracle.h.

All functions take and return numpy arrays.  Parity status: every function is
pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.oracle_histogram_u16.argtypes = [vp, u64, vp]
        L.oracle_histogram_u16.restype = None
        L.oracle_exclusive_scan_u64.argtypes = [vp, u64, vp]
        L.oracle_exclusive_scan_u64.restype = None
        L.oracle_reconstruct_counts_u16.argtypes = [vp, u64, u64, u64, vp]
        L.oracle_reconstruct_counts_u16.restype = None
        L.oracle_sort_u16.argtypes = [vp, u64, vp]
        L.oracle_sort_u16.restype = None
        L.oracle_trie_levels.argtypes = [vp, u64, i32, vp]
        L.oracle_trie_levels.restype = i32
        L.oracle_get_item.argtypes = [vp, i32, u64, u64]
        L.oracle_get_item.restype = u64
        L.oracle_get_index.argtypes = [vp, i32, u64]
        L.oracle_get_index.restype = u64
        L.oracle_bit_reverse.argtypes = [u64, i32]
        L.oracle_bit_reverse.restype = u64
        L.oracle_trie_depth.argtypes = [u64, i32]
        L.oracle_trie_depth.restype = i32
        L.oracle_decompose.argtypes = [u64, i32, i32, i32, vp, vp, vp]
        L.oracle_decompose.restype = None
        L.oracle_build_bins.argtypes = [vp, u64, i32, i32, i32, vp, vp]
        L.oracle_build_bins.restype = i32
        L.oracle_sort_bin.argtypes = [vp, u64, vp]
        L.oracle_sort_bin.restype = i32
        L.oracle_reconstruct_all.argtypes = [vp, vp, vp, i32, i32, i32, vp]
        L.oracle_reconstruct_all.restype = None
        L.oracle_trie_pack.argtypes = [vp, i32, u64, i32, vp, vp, vp, u64]
        L.oracle_trie_pack.restype = ctypes.c_int64
        L.oracle_counter_width.argtypes = [i32, u64, i32]
        L.oracle_counter_width.restype = i32
        L.oracle_alg5_sort.argtypes = [vp, u64, i32, i32, vp, vp]
        L.oracle_alg5_sort.restype = i32
        L.oracle_sort_pairs_u64_u32.argtypes = [vp, vp, u64, i32, vp, vp]
        L.oracle_sort_pairs_u64_u32.restype = i32
        L.oracle_sort_keys_u32.argtypes = [vp, u64, i32, vp]
        L.oracle_sort_keys_u32.restype = i32
        L.oracle_send_counts.argtypes = [vp, i32, i32, u64, vp]
        L.oracle_send_counts.restype = None
        L.oracle_check_nondecreasing_u16.argtypes = [vp, u64]
        L.oracle_check_nondecreasing_u16.restype = u64
        L.oracle_check_pairs_index.argtypes = [vp, u64, vp, vp]
        L.oracle_check_pairs_index.restype = u64
        L.oracle_sort_u16_mt.argtypes = [vp, u64, vp, i32]
        L.oracle_sort_u16_mt.restype = i32
        _lib = L
    return _lib


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray):
    return a.ctypes.data if a.size else None


def histogram_u16(keys) -> np.ndarray:
    k = _c(keys, np.uint16)
    C = np.empty(65536, dtype=np.uint64)
    lib().oracle_histogram_u16(_p(k), k.size, C.ctypes.data)
    return C


def exclusive_scan(C) -> np.ndarray:
    c = _c(C, np.uint64)
    P = np.empty(c.size + 1, dtype=np.uint64)
    lib().oracle_exclusive_scan_u64(_p(c), c.size, P.ctypes.data)
    return P


def reconstruct_counts_u16(C, out_begin=0, out_end=None) -> np.ndarray:
    c = _c(C, np.uint64)
    total = int(c.sum())
    out_end = total if out_end is None else out_end
    out = np.empty(max(0, out_end - out_begin), dtype=np.uint16)
    lib().oracle_reconstruct_counts_u16(_p(c), c.size, out_begin, out_end, _p(out))
    return out


def sort_u16(keys) -> np.ndarray:
    k = _c(keys, np.uint16)
    out = np.empty_like(k)
    lib().oracle_sort_u16(_p(k), k.size, _p(out))
    return out


def sort_u16_mt(keys, threads: int) -> np.ndarray:
    """The u16 oracle on `threads` POSIX threads (oracle_mt.c) -- timing only."""
    k = _c(keys, np.uint16)
    out = np.empty_like(k)
    rc = lib().oracle_sort_u16_mt(_p(k), k.size, _p(out), int(threads))
    if rc:
        raise RuntimeError(f"oracle_sort_u16_mt rc={rc}")
    return out


def trie_levels(keys, p) -> list:
    k = _c(keys, np.uint64)
    flat = np.empty((2 << p) - 1, dtype=np.uint64)
    rc = lib().oracle_trie_levels(_p(k), k.size, p, flat.ctypes.data)
    if rc:
        raise ValueError("oracle_trie_levels: p out of range")
    return [flat[(1 << l) - 1:(2 << l) - 1] for l in range(p + 1)]


def _flat(levels) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate(levels), dtype=np.uint64)


def get_item(levels, p, r, default=0) -> int:
    f = _flat(levels)
    return int(lib().oracle_get_item(f.ctypes.data, p, r, default))


def get_index(levels, p, v) -> int:
    f = _flat(levels)
    return int(lib().oracle_get_index(f.ctypes.data, p, v))


def bit_reverse(x, width) -> int:
    return int(lib().oracle_bit_reverse(x, width))


def trie_depth(n, p) -> int:
    return int(lib().oracle_trie_depth(n, p))


def decompose(key, p, l_n, l_b):
    b, o, t = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    lib().oracle_decompose(key, p, l_n, l_b, ctypes.byref(b), ctypes.byref(o), ctypes.byref(t))
    return b.value, o.value, t.value


def build_bins(keys, p, l_n, l_b):
    k = _c(keys, np.uint64)
    C = np.empty(1 << (l_n - l_b), dtype=np.uint64)
    E = np.empty(k.size, dtype=np.uint64)
    rc = lib().oracle_build_bins(_p(k), k.size, p, l_n, l_b, C.ctypes.data, _p(E))
    if rc:
        raise ValueError(f"oracle_build_bins rc={rc}")
    return C, E


def sort_bin(entries) -> np.ndarray:
    e = _c(entries, np.uint64)
    I = np.empty(e.size, dtype=np.uint64)
    rc = lib().oracle_sort_bin(_p(e), e.size, _p(I))
    if rc:
        raise ValueError(f"oracle_sort_bin rc={rc}")
    return I


def reconstruct_all(E, I, C, p, l_n, l_b) -> np.ndarray:
    e, i, c = _c(E, np.uint64), _c(I, np.uint64), _c(C, np.uint64)
    K = np.empty(e.size, dtype=np.uint64)
    lib().oracle_reconstruct_all(_p(e), _p(i), _p(c), p, l_n, l_b, _p(K))
    return K


def trie_pack(levels, p, capacity, min_width=1):
    """Tapered bit-packed export of the dense levels -> (widths, bit_offsets, packed words)."""
    f = _flat(levels)
    widths = np.zeros(p + 1, dtype=np.int32)
    offs = np.zeros(p + 2, dtype=np.uint64)
    words = ((1 << (p + 1)) * 64 + 63) // 64 + 1
    packed = np.zeros(words, dtype=np.uint64)
    used = lib().oracle_trie_pack(f.ctypes.data, p, capacity, min_width, widths.ctypes.data, offs.ctypes.data,
                                  packed.ctypes.data, words)
    if used < 0:
        raise ValueError("oracle_trie_pack: buffer too small")
    return widths, offs, packed[:used].copy()


def counter_width(level, capacity, min_width=1) -> int:
    return int(lib().oracle_counter_width(level, capacity, min_width))


def alg5_sort(keys, p, l_b):
    k = _c(keys, np.uint64)
    out = np.empty_like(k)
    n = k.size
    l_n = trie_depth(n, p)  # the C oracle's own l_n = min(p, ceil(log2 n)), pinned in the tests
    nb = 1 << (l_n - min(l_b, l_n))
    C = np.empty(nb, dtype=np.uint64)
    rc = lib().oracle_alg5_sort(_p(k), n, p, l_b, _p(out), C.ctypes.data)
    if rc:
        raise ValueError(f"oracle_alg5_sort rc={rc}")
    return out, C


def sort_pairs_u64_u32(keys, vals, key_bits=64):
    k = _c(keys, np.uint64)
    v = _c(vals, np.uint32) if vals is not None else None
    ko = np.empty_like(k)
    vo = np.empty_like(v) if v is not None else None
    rc = lib().oracle_sort_pairs_u64_u32(_p(k), _p(v) if v is not None else None, k.size, key_bits,
                                         _p(ko), _p(vo) if vo is not None else None)
    if rc:
        raise ValueError(f"oracle_sort_pairs_u64_u32 rc={rc}")
    return ko, vo


def sort_keys_u64(keys, key_bits=64):
    return sort_pairs_u64_u32(keys, None, key_bits)[0]


def sort_keys_u32(keys, key_bits=32):
    k = _c(keys, np.uint32)
    out = np.empty_like(k)
    rc = lib().oracle_sort_keys_u32(_p(k), k.size, key_bits, _p(out))
    if rc:
        raise ValueError(f"oracle_sort_keys_u32 rc={rc}")
    return out


def send_counts(C_all, g) -> np.ndarray:
    c = _c(C_all, np.uint64)
    G, nb = c.shape
    out = np.empty(G, dtype=np.uint64)
    lib().oracle_send_counts(c.ctypes.data, G, g, nb, out.ctypes.data)
    return out


def check_nondecreasing_u16(a) -> int:
    x = _c(a, np.uint16)
    return int(lib().oracle_check_nondecreasing_u16(_p(x), x.size))


def check_pairs_index(kin, kout, vout) -> int:
    a = _c(kin, np.uint64)
    b = _c(kout, np.uint64)
    c = _c(vout, np.uint32)
    return int(lib().oracle_check_pairs_index(_p(a), a.size, _p(b), _p(c)))
