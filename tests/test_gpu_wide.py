"""GPU parity of the multi-digit path (fs_sort_keys_u32/u64, fs_sort_pairs_u64_u32)
against the CPU oracle (stable LSD with 16-bit digits) and the four pair
invariants that pin the unique stable sort.  Bit-exact."""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2605_10390_b200 as fs

pytestmark = pytest.mark.gpu


def to_dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def to_host(t):
    return t.cpu().numpy()


SIZES = [1, 2, 31, 33, 4095, 4096, 4097, 100_003, (1 << 20) + 7]


@pytest.mark.parametrize("n", SIZES)
def test_sort_keys_u32(cuda, n):
    k = datagen.gen_u32(n, seed=n)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_keys_u32(k))


@pytest.mark.parametrize("n", SIZES)
def test_sort_keys_u64(cuda, n):
    k = datagen.gen_u64(n, seed=n)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_keys_u64(k))


@pytest.mark.parametrize("key_bits", [1, 7, 8, 9, 17, 33, 63, 64])
def test_sort_keys_u64_key_bits(cuda, key_bits):
    k = datagen.gen_u64(300_001, seed=key_bits, key_bits=key_bits)
    out = to_host(fs.sort_keys(to_dev(k, cuda), key_bits=key_bits))
    np.testing.assert_array_equal(out, oracle.sort_keys_u64(k, key_bits))


@pytest.mark.parametrize("n", SIZES)
def test_sort_pairs_uniform(cuda, n):
    k = datagen.gen_u64(n, seed=n + 1)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


@pytest.mark.parametrize("mask_bits", [0, 1, 4, 8, 12, 20])
def test_sort_pairs_low_entropy_stability(cuda, mask_bits):
    """Many equal keys: only a stable sort gives the oracle's value order."""
    n = 1_000_003
    k = datagen.gen_u64(n, seed=mask_bits) & np.uint64((1 << mask_bits) - 1)
    k = k | np.uint64(0xABCD000000000000)  # high digits constant: exercises skipped passes
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)
    assert oracle.check_pairs_index(k, to_host(ko), to_host(vo)) == 0


def test_sort_pairs_all_passes_skipped(cuda):
    n = 70_000
    k = np.full(n, 0x0123456789ABCDEF, dtype=np.uint64)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    np.testing.assert_array_equal(to_host(ko), k)
    np.testing.assert_array_equal(to_host(vo), v)


def test_c5_full_size_invariants(cuda):
    """Config c5 at full size (2^29 pairs) in bench.py's launch configuration:
    the four invariants pin the unique stable sort; a 2^22 prefix slice is also
    compared with the oracle element by element."""
    n = 1 << 29
    k = torch.empty(n, dtype=torch.uint64, device=cuda)
    v = torch.empty(n, dtype=torch.uint32, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
    datagen.iota_u32_device(v.data_ptr(), n, stream=s)
    ko, vo = fs.sort_pairs(k, v)
    kin = to_host(k)
    kout, vout = to_host(ko), to_host(vo)
    del ko, vo, k, v
    torch.cuda.empty_cache()
    assert oracle.check_pairs_index(kin, kout, vout) == 0
