"""The C-ABI boundary without a GPU: libfractalsort.so loads, exports every symbol
include/fractalsort.h declares, and rejects bad arguments before any CUDA call."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2605_10390_b200 as fs
from paper_2605_10390_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", src))
    return names


def test_header_and_binding_agree():
    decl = declared_functions()
    assert decl, "no declarations parsed"
    assert decl == set(_lib.SIGNATURES), decl ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = fs.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fs_[a-z0-9_]+)", out))
    assert declared_functions() <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version():
    L = fs.lib()
    assert L.fs_status_string(0) == b"FS_OK"
    assert L.fs_status_string(1) == b"FS_ERR_INVALID_ARGUMENT"
    assert L.fs_version() >> 16 == 1


V = ctypes.c_void_p


@pytest.mark.parametrize("call", [
    lambda L: L.fs_sort_keys_u16(None, None, 10, 0, None, 0, None),          # NULL with n > 0
    lambda L: L.fs_sort_keys_u16(V(0x1000), V(0x2000), 10, 17, V(0x100000), 1 << 30, None),  # key_bits
    lambda L: L.fs_sort_keys_u16(V(0x1000), V(0x2000), 10, 0, V(0x100000), 16, None),        # temp too small
    lambda L: L.fs_sort_keys_u16(V(0x1000), V(0x1002), 100, 0, V(0x1000000), 1 << 30, None),  # partial overlap
    lambda L: L.fs_sort_keys_u16(V(0x1000), V(0x4000), 10, 0, V(0x100010), 1 << 30, None),    # temp misaligned
    lambda L: L.fs_sort_keys_u64(V(0x1000), V(0x1000), 10, 0, V(0x1000000), 1 << 30, None),   # in == out
    lambda L: L.fs_sort_keys_u32(V(0x1000), V(0x8000), 10, 33, V(0x1000000), 1 << 30, None),  # key_bits
    lambda L: L.fs_sort_pairs_u64_u32(V(0x1000), None, V(0x9000), V(0xA000), 10, 0, V(0x1000000), 1 << 30, None),
    lambda L: L.fs_exclusive_scan_u64(V(0x1000), V(0x2000), 0, V(0x100000), 1 << 20, None),  # nbins 0
    lambda L: L.fs_exclusive_scan_u64(V(0x1000), V(0x1008), 16, V(0x100000), 1 << 20, None),  # overlap
    lambda L: L.fs_expand_u16(V(0x1000), 65537, 0, 10, V(0x8000), None),                     # nbins
    lambda L: L.fs_expand_u16(V(0x1000), 16, 10, 5, V(0x8000), None),                        # end < begin
    lambda L: L.fs_send_counts(V(0x1000), 2, 2, 16, V(0x8000), None),                         # g >= G
    lambda L: L.fs_histogram_u16(V(0x1000), 10, 0, None, 0, V(0x100000), 1 << 30, None),     # hist NULL
    lambda L: L.fs_sort_keys_u16_host(None, V(0x2000), 10, 0, V(0x100000), 1 << 30, None),
    lambda L: L.fs_trie_levels(V(0x1000), 25, V(0x100000), None),                             # p > 24
    lambda L: L.fs_trie_levels(V(0x1000), 4, V(0x1000), None),                                # overlap
    lambda L: L.fs_trie_pack(V(0x1000), 16, 100, 0, V(0x2000), V(0x3000), V(0x4000), 100, V(0x8000), 256, None),
    lambda L: L.fs_trie_pack(V(0x1000), 16, 100, 1, V(0x2000), V(0x3000), V(0x4000), 100, V(0x8000), 8, None),
    lambda L: L.fs_get_item(None, V(0x3000), V(0x4000), 16, V(0x5000), 4, 0, V(0x6000), None),
    lambda L: L.fs_get_index(V(0x2000), V(0x3000), V(0x4000), 0, V(0x5000), 4, V(0x6000), None),
    lambda L: L.fs_hist_merge_u64(V(0x1000), None, V(0x3000), 4, None),
    lambda L: L.fs_allreduce_multicast_u64(V(0x1000), V(0x9000), 4, None, V(0x5000), 1, 0, V(0x6000), None),  # flag
    lambda L: L.fs_allreduce_multicast_u64(V(0x1000), V(0x9000), 4, V(0x4002), V(0x5000), 1, 0, V(0x6000), None),
    lambda L: L.fs_allreduce_multicast_u64(V(0x1004), V(0x9000), 4, V(0x4000), V(0x5000), 1, 0, V(0x6000), None),
    lambda L: L.fs_allreduce_multicast_u64(V(0x1000), V(0x1008), 4, V(0x4000), V(0x5000), 1, 0, V(0x6000), None),
    lambda L: L.fs_allreduce_multicast_u64(None, V(0x9000), 4, V(0x4000), V(0x5000), 1, 0, V(0x6000), None),
    lambda L: L.fs_allreduce_multicast_u64(V(0x1000), V(0x9000), 4, V(0x4000), V(0x5000), 1, 0, None, None),  # timed_out
])
def test_invalid_arguments_rejected_without_gpu(call):
    L = fs.lib()
    assert call(L) == _lib.FS_ERR_INVALID_ARGUMENT
    assert L.fs_last_error_message()  # a detail string is set


def test_n_zero_is_ok_without_launch():
    L = fs.lib()
    assert L.fs_sort_keys_u16(None, None, 0, 0, None, 0, None) == _lib.FS_OK
    assert L.fs_sort_pairs_u64_u32(None, None, None, None, 0, 0, None, 0, None) == _lib.FS_OK
    assert L.fs_expand_u16(V(0x1000), 16, 7, 7, V(0x8000), None) == _lib.FS_OK
    assert L.fs_get_item(None, None, None, 16, None, 0, 0, None, None) == _lib.FS_OK
    assert L.fs_hist_merge_u64(None, None, None, 0, None) == _lib.FS_OK


def test_trie_sizes():
    L = fs.lib()
    assert L.fs_trie_levels_count(16) == (1 << 17) - 1
    assert L.fs_trie_levels_count(0) == 0
    # the word bound covers widths of bitlen(capacity) + 3 on every level
    assert L.fs_trie_pack_words(16, (1 << 28)) * 64 >= ((1 << 17) - 1) * 32
    assert L.fs_trie_pack_temp_bytes(16) >= 17 * 8


def test_temp_sizes_are_monotone_and_aligned():
    L = fs.lib()
    a, b = L.fs_sort_keys_u16_temp_bytes(1 << 20), L.fs_sort_keys_u16_temp_bytes(1 << 28)
    assert 0 < a <= b and b % 256 == 0
    assert L.fs_sort_pairs_u64_u32_temp_bytes(1 << 29, 64) >= (1 << 29) * 12
    assert L.fs_sort_keys_u64_temp_bytes(1000, 64) >= 8000


def test_cpu_tensors_fail_loudly():
    import torch
    with pytest.raises(ValueError):
        fs.sort_keys(torch.zeros(10, dtype=torch.uint16))


def test_multicast_allreduce_is_one_ldgmc_per_element():
    """fs_allreduce_multicast_u64's kernel reads through the switch: its SASS holds
    the multicast load-reduce (LDGMC ... ADD.64) and a system-scope RED for the
    barrier (checked here, on CPU, because the pool's one-GPU boxes have no
    NVSwitch multicast fabric to run it on: profiles/r02g/nvls_probe.txt)."""
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    fn = [blk for blk in sass.split("Function : ") if "k_allreduce_mc" in blk.split("\n", 1)[0]]
    assert len(fn) == 1
    assert "LDGMC.E.ADD.64" in fn[0]
    assert "REDG.E.ADD.STRONG.SYS" in fn[0]
