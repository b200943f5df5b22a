"""ctypes loader for libfractalsort.so (the C ABI declared in include/fractalsort.h).

Loading fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfractalsort.so")

FS_OK, FS_ERR_INVALID_ARGUMENT, FS_ERR_CUDA, FS_ERR_OUT_OF_MEMORY, FS_ERR_UNSUPPORTED = range(5)

_u64, _i32, _vp, _sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/fractalsort.h one to one.
SIGNATURES = {
    "fs_status_string": (ctypes.c_char_p, [_i32]),
    "fs_last_error_message": (ctypes.c_char_p, []),
    "fs_version": (_i32, []),
    "fs_sort_keys_u16_temp_bytes": (_sz, [_u64]),
    "fs_sort_keys_u32_temp_bytes": (_sz, [_u64, _i32]),
    "fs_sort_keys_u64_temp_bytes": (_sz, [_u64, _i32]),
    "fs_sort_pairs_u64_u32_temp_bytes": (_sz, [_u64, _i32]),
    "fs_histogram_u16_temp_bytes": (_sz, [_u64]),
    "fs_exclusive_scan_u64_temp_bytes": (_sz, [_u64]),
    "fs_sort_keys_u16": (_i32, [_vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "fs_sort_keys_u32": (_i32, [_vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "fs_sort_keys_u64": (_i32, [_vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "fs_sort_pairs_u64_u32": (_i32, [_vp, _vp, _vp, _vp, _u64, _i32, _vp, _sz, _vp]),
    "fs_histogram_u16": (_i32, [_vp, _u64, _i32, _vp, _i32, _vp, _sz, _vp]),
    "fs_exclusive_scan_u64": (_i32, [_vp, _vp, _u64, _vp, _sz, _vp]),
    "fs_histogram_prefix_u16": (_i32, [_vp, _u64, _vp, _vp, _sz, _vp]),
    "fs_expand_prefix_u16": (_i32, [_vp, _u64, _u64, _vp, _vp]),
    "fs_expand_u16": (_i32, [_vp, _u64, _u64, _u64, _vp, _vp]),
    "fs_send_counts": (_i32, [_vp, _i32, _i32, _u64, _vp, _vp]),
    "fs_sort_keys_u16_host_work_bytes": (_sz, [_u64, _u64]),
    "fs_sort_keys_u16_host": (_i32, [_vp, _vp, _u64, _u64, _vp, _sz, _vp]),
    "fs_set_phase_events": (_i32, [_vp, _i32]),
    "fs_bound_u64": (_i32, [_vp, _u64, _vp, _u64, _i32, _vp, _vp]),
    "fs_expand_to_peers_u16_temp_bytes": (_sz, [_u64, _i32]),
    "fs_expand_to_peers_u16": (_i32, [_vp, _i32, _i32, _u64, _vp, _vp, _sz, _vp]),
    "fs_allreduce_multicast_u64": (_i32, [_vp, _vp, _u64, _vp, _vp, ctypes.c_uint32, _u64, _vp, _vp]),
    "fs_trie_levels_count": (_sz, [_i32]),
    "fs_trie_levels": (_i32, [_vp, _i32, _vp, _vp]),
    "fs_trie_pack_words": (_sz, [_i32, _u64]),
    "fs_trie_pack_temp_bytes": (_sz, [_i32]),
    "fs_trie_pack": (_i32, [_vp, _i32, _u64, _i32, _vp, _vp, _vp, _u64, _vp, _sz, _vp]),
    "fs_get_item": (_i32, [_vp, _vp, _vp, _i32, _vp, _u64, _u64, _vp, _vp]),
    "fs_get_index": (_i32, [_vp, _vp, _vp, _i32, _vp, _u64, _vp, _vp]),
    "fs_hist_merge_u64": (_i32, [_vp, _vp, _vp, _u64, _vp]),
    "fs_histogram16_u64_temp_bytes": (_sz, [_u64]),
    "fs_histogram16_u64": (_i32, [_vp, _u64, _i32, _i32, _vp, _vp, _sz, _vp]),
    "fs_select_bins_u64": (_i32, [_vp, _u64, _i32, _i32, _vp, _i32, _vp, _u64, _vp, _vp]),
    "fs_digit_counts_sorted_u64": (_i32, [_vp, _u64, _vp, _i32, _i32, _i32, _vp, _vp]),
    "fs_pair_exchange_temp_bytes": (_sz, [_u64, _i32]),
    "fs_pair_classes_u64": (_i32, [_vp, _u64, _vp, _i32, _vp, _vp, _sz, _vp]),
    "fs_pair_scatter_u64_u32": (_i32, [_vp, _vp, _u64, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
}

_lib = None


class FractalSortError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)}: {detail}")


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension must be built (python -c "
                f"'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().fs_status_string(s).decode()


def check(status: int, where: str) -> None:
    if status != FS_OK:
        raise FractalSortError(status, where, lib().fs_last_error_message().decode())
