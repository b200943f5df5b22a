"""GPU parity of the order-statistic service through the
C ABI: dense trie levels from the GPU histogram vs the oracle's key-by-key Alg. 1
trie, the tapered bit-packed export vs oracle_trie_pack word for word, and batched
GetItem / GetIndex on the packed trie vs the oracle's Alg. 2 / Alg. 3 walks.
All integer: bit-exact."""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2605_10390_b200 as fs

pytestmark = pytest.mark.gpu


def _levels_flat(lv):
    return np.concatenate(lv).astype(np.uint64)


@pytest.mark.parametrize("dist,n,p", [("uniform", 100_003, 16), ("zipf", 300_001, 16), ("const", 5_000, 16),
                                      ("gauss", 77_777, 12), ("uniform", 1, 4), ("uniform", 0, 8)])
def test_levels_pack_and_queries(cuda, dist, n, p):
    keys = datagen.gen_u16(dist, n, seed=p).astype(np.uint16) >> np.uint16(16 - p)
    hist = fs.histogram_u16(torch.from_numpy(keys).to(cuda), key_bits=p)
    levels = fs.trie_levels(hist, p)
    lv = oracle.trie_levels(keys.astype(np.uint64), p)
    np.testing.assert_array_equal(levels.cpu().numpy().astype(np.uint64), _levels_flat(lv))

    t = fs.trie_pack(levels, p, max(n, 1), 2)
    w, off, words = oracle.trie_pack(lv, p, max(n, 1), 2)
    np.testing.assert_array_equal(t.widths.cpu().numpy(), w)
    np.testing.assert_array_equal(t.bit_offsets.cpu().numpy().astype(np.uint64), off)
    got = t.packed.cpu().numpy().astype(np.uint64)
    np.testing.assert_array_equal(got[:words.size], words)
    assert not got[words.size:].any()

    rng = np.random.default_rng(p + n)
    ranks = np.concatenate([rng.integers(0, max(n, 1) + 5, 4000), [0, max(n - 1, 0), n, n + 10**9]]).astype(np.uint64)
    items = fs.get_item(t, torch.from_numpy(ranks.astype(np.int64)).to(cuda), default=12345).cpu().numpy()
    want = [oracle.get_item(lv, p, int(r), 12345) for r in ranks]
    np.testing.assert_array_equal(items, np.array(want, dtype=np.int64))
    vals = np.concatenate([rng.integers(0, 1 << p, 4000), [0, (1 << p) - 1]]).astype(np.uint64)
    idx = fs.get_index(t, torch.from_numpy(vals.astype(np.int64)).to(cuda)).cpu().numpy()
    want = [oracle.get_index(lv, p, int(v)) for v in vals]
    np.testing.assert_array_equal(idx, np.array(want, dtype=np.int64))


def test_pack_buffer_too_small_flags_widths(cuda):
    p = 8
    keys = datagen.gen_u16("uniform", 10_000, seed=1) >> np.uint16(8)
    levels = fs.trie_levels(fs.histogram_u16(torch.from_numpy(keys).to(cuda), key_bits=p), p)
    # capacity far below the real total: the widths promote past the word bound
    t = fs.trie_pack(levels, p, capacity=1, min_width=1)
    assert int(t.widths[0].item()) == -1
    assert not t.packed.any().item()


def test_c2_quantiles_match_sorted_positions(cuda):
    """Config c2 at full size: quantiles from the packed trie equal the sorted
    output at the same ranks (the sort computed by the oracle at sampled ranks:
    rank r holds the v with P[v] <= r < P[v+1])."""
    n = 1 << 28
    k = torch.empty(n, dtype=torch.uint16, device=cuda)
    datagen.gen_u16_device(k.data_ptr(), "uniform", n, seed=0, stream=torch.cuda.current_stream().cuda_stream)
    hist = fs.histogram_u16(k)
    t = fs.trie_pack(fs.trie_levels(hist, 16), 16, n, 1)
    ranks = np.linspace(0, n - 1, 1001).astype(np.uint64)
    items = fs.get_item(t, torch.from_numpy(ranks.astype(np.int64)).to(cuda)).cpu().numpy()
    P = oracle.exclusive_scan(oracle.histogram_u16(k.cpu().numpy()))
    want = np.searchsorted(P, ranks, side="right") - 1
    np.testing.assert_array_equal(items, want)


def test_hist_merge_is_histogram_of_union(cuda):
    a = datagen.gen_u16("uniform", 50_000, seed=5)
    b = datagen.gen_u16("zipf", 70_000, seed=6)
    ha = fs.histogram_u16(torch.from_numpy(a).to(cuda))
    hb = fs.histogram_u16(torch.from_numpy(b).to(cuda))
    m = fs.hist_merge(ha, hb).cpu().numpy().astype(np.uint64)
    np.testing.assert_array_equal(m, oracle.histogram_u16(np.concatenate([a, b])))
