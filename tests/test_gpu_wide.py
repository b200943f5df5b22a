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
    the four invariants pin the unique stable sort; the first and last ~2^22
    outputs are also compared with the oracle element by element (the pairs whose
    key lies below 2^57 / at or above 2^64 - 2^57 are selected from the INPUT and
    sorted by the oracle; they must be exactly the head / tail of the output)."""
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
    idx = np.arange(n, dtype=np.uint32)
    for sel, where in ((kin < np.uint64(1 << 57), "head"), (kin >= np.uint64(2**64 - 2**57), "tail")):
        ek, ev = oracle.sort_pairs_u64_u32(kin[sel], idx[sel])
        m = ek.size
        assert (1 << 21) < m < (1 << 23)
        gk, gv = (kout[:m], vout[:m]) if where == "head" else (kout[n - m:], vout[n - m:])
        np.testing.assert_array_equal(gk, ek, err_msg=where)
        np.testing.assert_array_equal(gv, ev, err_msg=where)


# ---------------------------------------------------------------- trie-binned MSD path
# n >= 2^22 and key_bits >= 32 plan the MSD path (top-16 trie histogram, two
# stable 8-bit MSD scatters, per-bin local sort); the device falls back to LSD
# when a 16-bit bin exceeds the local-sort capacity.  Same oracle, bit-exact.
MSD_N = [1 << 22, (1 << 22) + 3, 5_000_011]


@pytest.mark.parametrize("n", MSD_N)
def test_msd_keys_u64(cuda, n):
    k = datagen.gen_u64(n, seed=n + 5)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_keys_u64(k))


@pytest.mark.parametrize("n", MSD_N)
def test_msd_keys_u32(cuda, n):
    k = datagen.gen_u32(n, seed=n + 6)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_keys_u32(k))


@pytest.mark.parametrize("n", MSD_N)
def test_msd_pairs(cuda, n):
    k = datagen.gen_u64(n, seed=n + 7)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


@pytest.mark.parametrize("key_bits", [32, 40, 48, 63])
def test_msd_pairs_key_bits(cuda, key_bits):
    n = (1 << 22) + 1
    k = datagen.gen_u64(n, seed=key_bits + 100, key_bits=key_bits)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda), key_bits=key_bits)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, key_bits)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


@pytest.mark.parametrize("distinct_low", [1, 2, 3, 40])
def test_msd_pairs_heavy_bins(cuda, distinct_low):
    """Bins that fit shared memory but hold long runs of equal keys: the local
    sort's slow path (stable LSD on the permutation) must keep arrival order."""
    n = 1 << 23  # 128 keys per 16-bit bin
    top = datagen.gen_u64(n, seed=11) & np.uint64(0xFFFF000000000000)
    low_vals = datagen.gen_u64(distinct_low, seed=12) & np.uint64((1 << 48) - 1)
    low = low_vals[datagen.gen_u64(n, seed=13) % np.uint64(distinct_low)]
    k = top | low
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


@pytest.mark.parametrize("bins", [256, 1500])
@pytest.mark.parametrize("copies", [2, 8, 16, 32, 64, 200])
def test_msd_pairs_repeated_keys(cuda, copies, bins):
    """Every key repeated ~`copies` times inside ~8,192-key 16-bit bins (256 bins
    used: k_local_sort) or ~1,400-key bins (1,500 used: k_local_mid): the per-bin
    group-size test sends a bin to the rank loop (groups <= kMaxGroup,
    key-weighted mean <= kMeanGroupMax) or to the slow path; with values =
    arrival indices, either must give the oracle's stable order."""
    n = 1 << 21
    tops = datagen.gen_u64(bins, seed=21) & np.uint64(0xFFFF000000000000)
    distinct = n // copies
    base = tops[datagen.gen_u64(distinct, seed=22) % np.uint64(bins)] | \
        (datagen.gen_u64(distinct, seed=23) & np.uint64((1 << 48) - 1))
    k = base[datagen.gen_u64(n, seed=24) % np.uint64(distinct)]
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("copies", [8, 64, 200])
def test_msd_keys_repeated(cuda, copies, width):
    """Keys-only sorts (fs_sort_keys_u32 / u64: the per-bin sort without values)
    of keys repeated ~`copies` times in ~8,192-key bins: rank loop, digit-first
    slow path with value sweeps, against the oracle."""
    n = 1 << 21
    if width == 64:
        tops = datagen.gen_u64(256, seed=41) & np.uint64(0xFFFF000000000000)
        distinct = n // copies
        base = tops[datagen.gen_u64(distinct, seed=42) % np.uint64(256)] | \
            (datagen.gen_u64(distinct, seed=43) & np.uint64((1 << 48) - 1))
        k = base[datagen.gen_u64(n, seed=44) % np.uint64(distinct)]
        want = oracle.sort_keys_u64(k)
    else:
        tops = datagen.gen_u32(256, seed=41) & np.uint32(0xFFFF0000)
        distinct = n // copies
        base = tops[datagen.gen_u32(distinct, seed=42) % np.uint32(256)] | \
            (datagen.gen_u32(distinct, seed=43) & np.uint32(0xFFFF))
        k = base[datagen.gen_u32(n, seed=44) % np.uint32(distinct)]
        want = oracle.sort_keys_u32(k)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), want)


@pytest.mark.parametrize("low_values", [1, 3, 16, 17, 0])
def test_msd_pairs_slow_path_groups(cuda, low_values):
    """~8,192-key bins whose keys share the counting digit (the 12 bits below the
    16-bit bin) and differ only in the low 36 bits: every bin is one group, so it
    takes the slow path; it sorts by the counting digit first, then finishes a
    group of <= 16 distinct keys by stable value sweeps (1, 3, 16 values) or
    falls back to the full LSD (17 values; 0 = all-random low bits)."""
    n = 1 << 21
    tops = datagen.gen_u64(256, seed=31) & np.uint64(0xFFFFFFF000000000)
    top = tops[datagen.gen_u64(n, seed=32) % np.uint64(256)]
    rnd = datagen.gen_u64(n, seed=33) & np.uint64((1 << 36) - 1)
    if low_values:
        vals = datagen.gen_u64(low_values, seed=34) & np.uint64((1 << 36) - 1)
        rnd = vals[datagen.gen_u64(n, seed=35) % np.uint64(low_values)]
    k = top | rnd
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


def _check_pairs(cuda, k, key_bits=64):
    v = datagen.iota_u32(len(k))
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda), key_bits=key_bits)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, key_bits)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda), key_bits=key_bits)), ek)


def test_msd_recursion_one_oversize_bin(cuda):
    """One 16-bit bin above the local-sort capacity: it recurses on the next
    digit while the other bins take the local sort."""
    n = (1 << 22) + 9
    k = datagen.gen_u64(n, seed=21)
    k[: 20_000] = (k[: 20_000] & np.uint64((1 << 48) - 1)) | np.uint64(0x1234 << 48)
    _check_pairs(cuda, k)


@pytest.mark.parametrize("nhot", [1, 3, 64])
def test_msd_recursion_many_oversize_bins(cuda, nhot):
    """Half the keys in `nhot` hot 16-bit bins (one level of recursion splits
    them), the rest spread over all bins."""
    n = (1 << 22) + 13
    k = datagen.gen_u64(n, seed=40 + nhot)
    hot = datagen.gen_u64(n, seed=41) % np.uint64(2) == 0
    tops = datagen.gen_u64(nhot, seed=42) >> np.uint64(48)
    pick = tops[datagen.gen_u64(n, seed=43) % np.uint64(nhot)]
    k[hot] = (k[hot] & np.uint64((1 << 48) - 1)) | (pick[hot] << np.uint64(48))
    _check_pairs(cuda, k)


def test_msd_recursion_deep(cuda):
    """Hot bins whose next 16 bits are concentrated too: the recursion goes
    several digits down before the pieces fit, with duplicate keys at the bottom."""
    n = (1 << 22) + 3
    k = datagen.gen_u64(n, seed=50)
    sel = datagen.gen_u64(n, seed=51)
    hot = sel % np.uint64(4) != 0
    a = np.array([0x0001, 0xBEEF, 0x7F00], dtype=np.uint64)[sel % np.uint64(3)]
    b = np.array([0x0000, 0x00FF, 0xFF00, 0x8001], dtype=np.uint64)[(sel >> np.uint64(8)) % np.uint64(4)]
    low = (sel >> np.uint64(16)) % np.uint64(5000)  # many duplicates
    k[hot] = (a[hot] << np.uint64(48)) | (b[hot] << np.uint64(32)) | low[hot]
    _check_pairs(cuda, k)


def test_msd_recursion_equal_keys(cuda):
    """Oversize bins of equal keys: one that never moves (every digit uniform)
    and one split once, whose halves then stay in the temporary buffer and are
    copied out at the last level."""
    n = (1 << 22) + 1
    k = datagen.gen_u64(n, seed=60)
    k[:30_000] = np.uint64(0xABCD_0123_4567_89AB)
    k[30_000:60_000] = np.uint64(0x5555_1000_0000_0001)
    k[60_000:90_000] = np.uint64(0x5555_2000_0000_0001)
    k = k[datagen.gen_u64(n, seed=61).argsort(kind="stable")]
    _check_pairs(cuda, k)


@pytest.mark.parametrize("key_bits", [32, 37, 40, 48])
def test_msd_recursion_key_bits(cuda, key_bits):
    """Oversize bins at narrower key widths (the last digit shorter than 8 bits
    when key_bits - 16 is not a multiple of 8); u32 keys too."""
    n = (1 << 22) + 7
    k = datagen.gen_u64(n, seed=70 + key_bits, key_bits=key_bits)
    hot = datagen.gen_u64(n, seed=71) % np.uint64(3) == 0
    k[hot] = (k[hot] & np.uint64((1 << (key_bits - 16)) - 1)) | np.uint64(0x00C3 << (key_bits - 16))
    _check_pairs(cuda, k, key_bits)
    if key_bits <= 32:
        k32 = k.astype(np.uint32)
        np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k32, cuda), key_bits=key_bits)),
                                      oracle.sort_keys_u32(k32, key_bits))


def test_msd_recursion_unaligned_buffers(cuda):
    """Oversize bins and uneven first-level buckets with buffers that are not
    16-byte aligned: k_heavy loads its tiles without bulk copies."""
    n = (1 << 22) + 11
    k = datagen.gen_u64(n + 1, seed=90)
    hot = datagen.gen_u64(n + 1, seed=91) % np.uint64(5) < np.uint64(2)
    k[hot] = (k[hot] & np.uint64((1 << 48) - 1)) | np.uint64(0x9ABC << 48)
    v = datagen.iota_u32(n + 1)
    kd, vd = to_dev(k, cuda)[1:], to_dev(v, cuda)[1:]
    ko, vo = fs.sort_pairs(kd, vd)
    ek, ev = oracle.sort_pairs_u64_u32(k[1:], v[1:])
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


def test_msd_recursion_many_small_oversize_bins(cuda):
    """Hundreds of bins just above the capacity (8,705 to 9,000 keys): one chunk
    per segment, sub-bins merged into items."""
    n = (1 << 22) + 2
    k = datagen.gen_u64(n, seed=95)
    nb = 400
    sizes = 8705 + (datagen.gen_u64(nb, seed=96) % np.uint64(296)).astype(np.int64)
    tops = (np.arange(nb, dtype=np.uint64) * np.uint64(163)) << np.uint64(48)
    pos = 0
    for t, m in zip(tops, sizes):
        k[pos:pos + m] = (k[pos:pos + m] & np.uint64((1 << 48) - 1)) | t
        pos += int(m)
    k = k[datagen.gen_u64(n, seed=97).argsort(kind="stable")]
    _check_pairs(cuda, k)


@pytest.mark.parametrize("prefix,free_bits", [(0, 40), (0xABCDEF, 40), (0, 32), (0x5A, 56), (1, 63)])
def test_msd_common_prefix_window(cuda, prefix, free_bits):
    """Keys sharing their bits above `free_bits` (a common prefix, zero or not):
    the MSD path bins the 16 bits below the prefix (a rebuilt trie histogram)
    and puts the prefix back on every key."""
    n = (1 << 22) + 5
    k = datagen.gen_u64(n, seed=80 + free_bits) & np.uint64((1 << free_bits) - 1)
    k |= np.uint64(prefix) << np.uint64(free_bits)
    _check_pairs(cuda, k)


def test_msd_common_prefix_with_oversize_bins(cuda):
    """A common prefix and, below it, oversize bins: the recursion runs on the
    shifted window."""
    n = (1 << 22) + 5
    k = datagen.gen_u64(n, seed=85) & np.uint64((1 << 44) - 1)
    hot = datagen.gen_u64(n, seed=86) % np.uint64(4) == 0
    k[hot] = (k[hot] & np.uint64((1 << 28) - 1)) | np.uint64(0xBEE << 28)
    k |= np.uint64(0x77) << np.uint64(48)
    _check_pairs(cuda, k)


def test_msd_narrow_effective_keys_take_lsd(cuda):
    """Fewer than 32 varying bits under key_bits = 64: the LSD path (uniform
    digits skipped)."""
    n = (1 << 22) + 5
    k = datagen.gen_u64(n, seed=87) & np.uint64((1 << 24) - 1)
    _check_pairs(cuda, k)


@pytest.mark.parametrize("n", [8_961, 16_384, (1 << 15) - 1, 1 << 15, 50_001, 1 << 18, 700_001, (1 << 21) + 5])
@pytest.mark.parametrize("kind", ["uniform", "few", "sorted"])
def test_msd_small_inputs(cuda, n, kind):
    """MSD from 8,961 pairs: bins of <= 128 keys sorted by one warp each
    (k_tiny_bins), the others by k_local_sort from the plan's list; ties among
    duplicates keep arrival order."""
    k = datagen.gen_u64(n, seed=n % 1013)
    if kind == "few":  # ~16 keys per distinct value: tiny bins full of ties
        k = k[datagen.gen_u64(n, seed=3) % np.uint64(max(1, n // 16))]
    elif kind == "sorted":
        k = np.sort(k)
    _check_pairs(cuda, k)


@pytest.mark.parametrize("n", [1, 2, 777, 8192, 8_960, 8_961, 10_241, 16383, 16384, 16385])
@pytest.mark.parametrize("key_bits", [13, 31, 32, 64])
def test_small_single_cta_sort(cuda, n, key_bits):
    """n <= 8,960 (<= 16,384 with key_bits < 32): the whole LSD in one CTA's shared
    memory (k_small_sort), incl. digits skipped because every key shares them;
    above, the multi-kernel paths (MSD, or LSD-8 for key_bits < 32)."""
    k = datagen.gen_u64(n, seed=n + key_bits, key_bits=key_bits)
    _check_pairs(cuda, k, key_bits)
    if key_bits <= 32:
        k32 = k.astype(np.uint32)
        np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k32, cuda), key_bits=key_bits)),
                                      oracle.sort_keys_u32(k32, key_bits))


def test_small_single_cta_sort_equal_and_few(cuda):
    """All keys equal (no pass runs: output = input order) and few distinct keys."""
    k = np.full(5000, 0xDEADBEEF, dtype=np.uint64)
    _check_pairs(cuda, k)
    k = datagen.gen_u64(3, seed=4)[datagen.gen_u64(6000, seed=5) % np.uint64(3)]
    _check_pairs(cuda, k)


def test_msd_unaligned_buffers(cuda):
    """Inputs/outputs not 16-byte aligned: the scatter passes load tiles without bulk copies."""
    n = (1 << 22) + 5
    k = datagen.gen_u64(n + 1, seed=31)
    v = datagen.iota_u32(n + 1)
    kd, vd = to_dev(k, cuda)[1:], to_dev(v, cuda)[1:]
    ko, vo = fs.sort_pairs(kd, vd)
    ek, ev = oracle.sort_pairs_u64_u32(k[1:], v[1:])
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


def _fuzz_keys(rng, n, key_bits, kind):
    k = datagen.gen_u64(n, seed=int(rng.integers(1 << 30)), key_bits=key_bits)
    if kind == "few":          # a handful of distinct values
        vals = datagen.gen_u64(7, seed=int(rng.integers(1 << 30)), key_bits=key_bits)
        k = vals[k % np.uint64(7)]
    elif kind == "sorted":
        k = np.sort(k)
    elif kind == "reverse":
        k = np.sort(k)[::-1].copy()
    elif kind == "lowbits":    # only the low 20 bits vary
        k = (k & np.uint64((1 << min(20, key_bits)) - 1)) | (np.uint64(0xABCDEF) << np.uint64(max(0, key_bits - 24))
                                                             if key_bits > 24 else np.uint64(0))
        if key_bits < 64:
            k &= np.uint64((1 << key_bits) - 1)
    elif kind == "bincap":     # top-16 bins right at the local-sort capacity (8,704)
        top = (np.arange(n, dtype=np.uint64) // np.uint64(8704)) << np.uint64(key_bits - 16)
        k = top | (k & np.uint64((1 << (key_bits - 16)) - 1))
        k = k[rng.permutation(n)]
    return k


@pytest.mark.parametrize("case", range(16))
def test_fuzz_pairs_and_keys(cuda, case):
    """Random sizes around the MSD threshold, key widths and adversarial shapes
    (few distinct values, sorted, reverse, low-entropy, bins exactly at the
    local-sort capacity) through all three wide entry points; oracle, bit-exact."""
    rng = np.random.default_rng(1000 + case)
    kinds = ["uniform", "few", "sorted", "reverse", "lowbits", "bincap"]
    kind = kinds[case % len(kinds)]
    key_bits = int(rng.choice([32, 37, 48, 56, 64])) if kind != "bincap" else 64
    n = int(rng.integers((1 << 22) - 1000, 3 * (1 << 21))) if case % 2 == 0 else int(rng.integers(1, 300_000))
    k = _fuzz_keys(rng, n, key_bits, kind)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda), key_bits=key_bits)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, key_bits)
    np.testing.assert_array_equal(to_host(ko), ek, err_msg=f"{kind} n={n} kb={key_bits}")
    np.testing.assert_array_equal(to_host(vo), ev, err_msg=f"{kind} n={n} kb={key_bits}")
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda), key_bits=key_bits)), ek)
    if key_bits <= 32:
        k32 = k.astype(np.uint32)
        np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k32, cuda), key_bits=key_bits)),
                                      oracle.sort_keys_u32(k32, key_bits))


def test_msd_level2_linear_order(cuda):
    """A first-level bucket holding 30% of the keys (bins still fit the local
    sort): 256 x (its tiles) exceeds the status rows, so level 2 is not run by
    the interleaved k_scatter but by k_heavy over the buckets as segments
    (per-chunk digit histograms, CTA-owned chunks, no lookback)."""
    n = (1 << 22) + 5
    k = datagen.gen_u64(n, seed=77)
    hot = datagen.gen_u64(n, seed=78) % np.uint64(10) < np.uint64(3)
    k[hot] = (k[hot] & np.uint64((1 << 56) - 1)) | np.uint64(0x42 << 56)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(ko), ek)
    np.testing.assert_array_equal(to_host(vo), ev)


def test_concurrent_streams(cuda):
    """Sorts on two CUDA streams at once (one-cluster u16, two-kernel u16, MSD
    pairs with an oversize bin, u32 keys): the library keeps no state between
    calls, so concurrent calls with their own temporaries do not interfere."""
    a16 = datagen.gen_u16("zipf", 200_003, seed=1)
    b16 = datagen.gen_u16("uniform", (1 << 22) + 1, seed=2)
    k = datagen.gen_u64((1 << 21) + 3, seed=3)
    k[:20_000] = (k[:20_000] & np.uint64((1 << 48) - 1)) | np.uint64(0x3333 << 48)
    v = datagen.iota_u32(k.size)
    k32 = datagen.gen_u32(3_000_001, seed=4)
    da, db, dk, dv, d32 = (to_dev(x, cuda) for x in (a16, b16, k, v, k32))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(device=cuda), torch.cuda.Stream(device=cuda)
    for _ in range(3):
        with torch.cuda.stream(s1):
            ra = fs.sort_keys(da)
            rk, rv = fs.sort_pairs(dk, dv)
        with torch.cuda.stream(s2):
            rb = fs.sort_keys(db)
            r32 = fs.sort_keys(d32)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(ra), oracle.sort_u16(a16))
    np.testing.assert_array_equal(to_host(rb), oracle.sort_u16(b16))
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(to_host(rk), ek)
    np.testing.assert_array_equal(to_host(rv), ev)
    np.testing.assert_array_equal(to_host(r32), oracle.sort_keys_u32(k32))


def _fuzz_shape(rng, n):
    """A random mixture: uniform keys, a common prefix, hot 16-bit bins, few
    distinct values, sorted runs — so sizes and shapes cross every path (one-CTA
    LSD, LSD-8, MSD with tiny / mid / large bins, recursion, moved window)."""
    kb = int(rng.choice([24, 32, 40, 48, 56, 64]))
    k = datagen.gen_u64(n, seed=int(rng.integers(1 << 30)), key_bits=kb)
    shape = int(rng.integers(6))
    if shape == 1 and kb > 20:  # common prefix above a random bit
        free = int(rng.integers(8, kb))
        k = (k & np.uint64((1 << free) - 1)) | np.uint64(int(rng.integers(1, 1 << (kb - free))) << free
                                                       if kb - free < 63 else 0)
    elif shape == 2:  # hot bins
        sel = datagen.gen_u64(n, seed=int(rng.integers(1 << 30))) % np.uint64(3) == 0
        hot = datagen.gen_u64(int(rng.integers(1, 20)), seed=int(rng.integers(1 << 30)), key_bits=kb)
        k[sel] = hot[datagen.gen_u64(int(sel.sum()), seed=7) % np.uint64(hot.size)] ^ (k[sel] & np.uint64(0xFFF))
    elif shape == 3:  # few distinct values
        vals = datagen.gen_u64(int(rng.integers(1, 50)), seed=int(rng.integers(1 << 30)), key_bits=kb)
        k = vals[k % np.uint64(vals.size)]
    elif shape == 4:  # sorted runs with noise
        k = np.sort(k)
        k[::97] = datagen.gen_u64(k[::97].size, seed=9, key_bits=kb)
    if kb < 64:
        k &= np.uint64((1 << kb) - 1)
    return k, kb


@pytest.mark.parametrize("case", range(24))
def test_fuzz_every_path(cuda, case):
    rng = np.random.default_rng(5000 + case)
    lo = 0 if case % 2 else np.log(20_000)  # every other case at least 20,000 keys
    n = int(np.exp(rng.uniform(lo, np.log(6_000_000))))
    k, kb = _fuzz_shape(rng, n)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(to_dev(k, cuda), to_dev(v, cuda), key_bits=kb)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, kb)
    np.testing.assert_array_equal(to_host(ko), ek, err_msg=f"n={n} kb={kb}")
    np.testing.assert_array_equal(to_host(vo), ev, err_msg=f"n={n} kb={kb}")


# ---------------------------------------------------------------- maximum sizes
# Inputs far above c5, checked on the device (a host copy of 24-32 GB would take
# minutes) by the invariants that pin the unique result: output sorted; values a
# permutation of 0..n-1 with keys[values] == sorted keys and increasing within
# equal keys (pairs); per-top-16-bit counts and the key sum preserved (keys).
# At 2^31 pairs every 16-bit bin (~32,768 pairs) exceeds the local-sort
# capacity, so the whole input goes through the recursion (k_heavy).
_SIGN = torch.iinfo(torch.int64).min
_CHUNK = 1 << 28


def _sorted_chunked(x64):
    prev = None
    for c0 in range(0, x64.numel(), _CHUNK):
        b = x64[c0:c0 + _CHUNK]
        if not bool((b[1:] >= b[:-1]).all().item()) or (prev is not None and not bool((b[0] >= prev).item())):
            return False
        prev = b[-1]
    return True


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_max_size_pairs_2_31(cuda):
    _free()
    n = 1 << 31
    s = torch.cuda.current_stream().cuda_stream
    k = torch.empty(n, dtype=torch.uint64, device=cuda)
    v = torch.empty(n, dtype=torch.uint32, device=cuda)
    datagen.gen_u64_device(k.data_ptr(), n, seed=3, stream=s)
    datagen.iota_u32_device(v.data_ptr(), n, stream=s)
    ko, vo = fs.sort_pairs(k, v)
    del v
    ko64 = ko.view(torch.int64)
    assert _sorted_chunked(ko64 ^ _SIGN)
    idx = vo.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    del vo
    mark = torch.zeros(n, dtype=torch.uint8, device=cuda)
    mark[idx] = 1
    assert bool(mark.all().item())
    del mark
    assert bool((k.view(torch.int64)[idx] == ko64).all().item())
    same = ko64[1:] == ko64[:-1]
    assert bool((~same | (idx[1:] > idx[:-1])).all().item())
    del k, ko, ko64, idx, same
    _free()


@pytest.mark.parametrize("dt", [torch.uint32, torch.uint64])
def test_max_size_keys_2_32(cuda, dt):
    """n = 2^32 keys: element counts past 32 bits everywhere on the path."""
    _free()
    n = 1 << 32
    s = torch.cuda.current_stream().cuda_stream
    k = torch.empty(n, dtype=dt, device=cuda)
    (datagen.gen_u32_device if dt == torch.uint32 else datagen.gen_u64_device)(k.data_ptr(), n, seed=5, stream=s)
    out = fs.sort_keys(k)
    hk = torch.zeros(65536, dtype=torch.int64, device=cuda)
    ho = torch.zeros_like(hk)
    sk = so = 0
    prev = None
    for c0 in range(0, n, _CHUNK):
        if dt == torch.uint32:
            a = k[c0:c0 + _CHUNK].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            b = out[c0:c0 + _CHUNK].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            sh = 16
        else:
            a = k[c0:c0 + _CHUNK].view(torch.int64) ^ _SIGN
            b = out[c0:c0 + _CHUNK].view(torch.int64) ^ _SIGN
            sh = 48
        assert bool((b[1:] >= b[:-1]).all().item())
        assert prev is None or bool((b[0] >= prev).item())
        prev = b[-1]
        hk += torch.bincount((a >> sh) & 0xFFFF, minlength=65536)
        ho += torch.bincount((b >> sh) & 0xFFFF, minlength=65536)
        sk += int((a & 0xFFFFFFF).sum().item())
        so += int((b & 0xFFFFFFF).sum().item())
    assert bool((hk == ho).all().item()) and sk == so
    del k, out, a, b
    _free()
