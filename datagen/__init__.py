"""Seeded synthetic inputs for tests/, bench.py and smoke().

TEST/BENCH INFRASTRUCTURE.  This module is shared by the oracle side and the
CUDA side of the parity tests and holds none of the sorting method's
arithmetic: it only maps (distribution, seed, global index) to a key.  The
recipes are documented in datagen/datagen.cu and DESIGN.md §Inputs.

Host generators return numpy arrays; device generators fill caller-owned device
memory (raw pointers, e.g. ``tensor.data_ptr()``) on a given CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfsdatagen.so")

UNIFORM, ZIPF, GAUSS, SORTEDSWAP, CONST = 0, 1, 2, 3, 4
DISTS = {"uniform": UNIFORM, "zipf": ZIPF, "gauss": GAUSS, "sortedswap": SORTEDSWAP, "const": CONST}
CONST_KEY = 0xA5A5  # SURVEY.md §8(c).3 ledger 22: "all keys equal" uses 42,405

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build() (make -C {os.path.dirname(_HERE)})")
        L = ctypes.CDLL(_LIB_PATH)
        u64, i32, u32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        L.fsg_gen_u16_host.argtypes = [i32, u64, u64, u64, u64, i32, u32, vp]
        L.fsg_gen_u16_device.argtypes = [i32, u64, u64, u64, u64, i32, u32, vp, vp]
        L.fsg_gen_u32_host.argtypes = [u64, u64, u64, i32, vp]
        L.fsg_gen_u64_host.argtypes = [u64, u64, u64, i32, vp]
        L.fsg_gen_u32_device.argtypes = [u64, u64, u64, i32, vp, vp]
        L.fsg_gen_u64_device.argtypes = [u64, u64, u64, i32, vp, vp]
        L.fsg_iota_u32_host.argtypes = [u64, u64, vp]
        L.fsg_iota_u32_device.argtypes = [u64, u64, vp, vp]
        L.fsg_tables.argtypes = [i32, u64, vp, vp, vp]
        for f in ("fsg_gen_u16_host", "fsg_gen_u16_device", "fsg_gen_u32_host", "fsg_gen_u64_host",
                  "fsg_gen_u32_device", "fsg_gen_u64_device", "fsg_iota_u32_host", "fsg_iota_u32_device",
                  "fsg_tables"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")


def _dist_id(dist) -> int:
    return DISTS[dist] if isinstance(dist, str) else int(dist)


def gen_u16(dist="uniform", n=0, seed=0, i0=0, n_total=None, key_bits=16, param=CONST_KEY) -> np.ndarray:
    """Host u16 keys [i0, i0+n) of an n_total-key input."""
    n_total = n if n_total is None else n_total
    out = np.empty(n, dtype=np.uint16)
    _check(lib().fsg_gen_u16_host(_dist_id(dist), seed, i0, n, n_total, key_bits, param,
                                  out.ctypes.data), "fsg_gen_u16_host")
    return out


def gen_u16_device(out_ptr: int, dist="uniform", n=0, seed=0, i0=0, n_total=None, key_bits=16,
                   param=CONST_KEY, stream=0) -> None:
    n_total = n if n_total is None else n_total
    _check(lib().fsg_gen_u16_device(_dist_id(dist), seed, i0, n, n_total, key_bits, param, out_ptr, stream),
           "fsg_gen_u16_device")


def gen_u32(n, seed=0, i0=0, key_bits=32) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _check(lib().fsg_gen_u32_host(seed, i0, n, key_bits, out.ctypes.data), "fsg_gen_u32_host")
    return out


def gen_u64(n, seed=0, i0=0, key_bits=64) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    _check(lib().fsg_gen_u64_host(seed, i0, n, key_bits, out.ctypes.data), "fsg_gen_u64_host")
    return out


def gen_u32_device(out_ptr, n, seed=0, i0=0, key_bits=32, stream=0) -> None:
    _check(lib().fsg_gen_u32_device(seed, i0, n, key_bits, out_ptr, stream), "fsg_gen_u32_device")


def gen_u64_device(out_ptr, n, seed=0, i0=0, key_bits=64, stream=0) -> None:
    _check(lib().fsg_gen_u64_device(seed, i0, n, key_bits, out_ptr, stream), "fsg_gen_u64_device")


def iota_u32(n, i0=0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _check(lib().fsg_iota_u32_host(i0, n, out.ctypes.data), "fsg_iota_u32_host")
    return out


def iota_u32_device(out_ptr, n, i0=0, stream=0) -> None:
    _check(lib().fsg_iota_u32_device(i0, n, out_ptr, stream), "fsg_iota_u32_device")


def tables(dist, seed=0):
    T = np.empty(65536, dtype=np.uint64)
    G = np.empty(65536, dtype=np.uint32)
    P = np.empty(65536, dtype=np.uint16)
    _check(lib().fsg_tables(_dist_id(dist), seed, T.ctypes.data, G.ctypes.data, P.ctypes.data), "fsg_tables")
    return T, G, P
