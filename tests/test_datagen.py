"""The seeded synthetic inputs (ledger 18-22): determinism, frozen
golden hashes, sharding by global index, and the distribution shapes the configs
name (Zipf s=1.2 top value ~19.8%, Gaussian N(32768, 1024), sorted + 1% swaps)."""
import hashlib
import json
import os

import numpy as np

import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "datagen_first1024.json")))


def sha(a):
    return hashlib.sha256(a.tobytes()).hexdigest()


def test_golden_hashes():
    for d in ["uniform", "zipf", "gauss", "const"]:
        a = datagen.gen_u16(d, 1024, seed=0, n_total=1 << 28)
        assert sha(a) == GOLD[f"u16_{d}"]["sha256"], d
    assert sha(datagen.gen_u16("sortedswap", 1 << 20, seed=0)[:1024]) == GOLD["u16_sortedswap_n2^20"]["sha256"]
    assert sha(datagen.gen_u64(1024, seed=0)) == GOLD["u64_uniform"]["sha256"]
    assert sha(datagen.gen_u32(1024, seed=0)) == GOLD["u32_uniform"]["sha256"]


def test_determinism_and_seed_sensitivity():
    for d in ["uniform", "zipf", "gauss", "sortedswap"]:
        a = datagen.gen_u16(d, 100_000, seed=3)
        assert np.array_equal(a, datagen.gen_u16(d, 100_000, seed=3))
        assert not np.array_equal(a, datagen.gen_u16(d, 100_000, seed=4))


def test_sharding_by_global_index():
    n = 1_000_000
    full = datagen.gen_u16("zipf", n, seed=1)
    parts = [datagen.gen_u16("zipf", n // 4, seed=1, i0=g * n // 4, n_total=n) for g in range(4)]
    assert np.array_equal(np.concatenate(parts), full)
    f64 = datagen.gen_u64(n, seed=2)
    assert np.array_equal(np.concatenate([datagen.gen_u64(n // 2, seed=2, i0=g * n // 2) for g in range(2)]), f64)


def test_zipf_shape():
    n = 1 << 22
    k = datagen.gen_u16("zipf", n, seed=0)
    c = np.sort(np.bincount(k, minlength=65536))[::-1]
    H = sum(r ** -1.2 for r in range(1, 65537))
    assert abs(c[0] / n - 1 / H) < 0.002            # P(rank 1) = 1/H = 0.198
    assert abs(c[1] / n - 2 ** -1.2 / H) < 0.002
    assert c[0] >= 100 * n / 65536                   # >= 100x uniform expectation
    T, G, P = datagen.tables("zipf", 0)
    assert np.all(np.diff(T.astype(object)) >= 0) and T[-1] == np.iinfo(np.uint64).max
    assert sorted(P.tolist()) == list(range(65536))  # the value permutation is a permutation


def test_gauss_shape():
    k = datagen.gen_u16("gauss", 1 << 22, seed=0).astype(np.float64)
    assert abs(k.mean() - 32768) < 2 and abs(k.std() - 1024) < 2


def test_sortedswap_shape():
    n = 1 << 20
    k = datagen.gen_u16("sortedswap", n, seed=0)
    base = ((np.arange(n, dtype=np.uint64) * 65536) // n).astype(np.uint16)
    moved = int((k != base).sum())
    assert 0 < moved <= 2 * (n // 100)
    assert np.array_equal(np.bincount(k, minlength=65536), np.bincount(base, minlength=65536))


def test_uniform_key_bits_and_iota():
    k = datagen.gen_u16("uniform", 100_000, key_bits=5)
    assert k.max() < 32 and len(np.unique(k)) == 32
    k = datagen.gen_u64(100_000, key_bits=17)
    assert int(k.max()) < (1 << 17)
    assert np.array_equal(datagen.iota_u32(10, i0=5), np.arange(5, 15, dtype=np.uint32))
