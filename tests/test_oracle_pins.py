"""Pins of the CPU oracle to things other than itself (CPU only, -m "not gpu").

Each test pins oracle functions to one of: the worked examples printed in
SPEC.md / PAPER.md (tests/golden/spec_examples.json, cited per entry), exhaustive
brute force on tiny inputs, library routines that compute the same plain
definition (Python sorted(), numpy sort / argsort(kind='stable') / bincount /
cumsum / searchsorted), closed forms, and invariants (conservation, sibling sum,
permutation, stability).  Chosen so that a dropped term, wrong sign or index, or
transposed operand in the oracle fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest

import datagen
import oracle
from paper_2605_10390_b200 import metrics

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------- SPEC/PAPER worked examples
def test_golden_insert_5_1_5():
    g = GOLD["insert_5_1_5"]
    lv = oracle.trie_levels(np.array(g["keys"]), g["p"])
    assert lv[0][0] == g["root"]
    assert lv[1][1] == g["level1_bit1"] and lv[1][0] == g["level1_bit0"]
    assert lv[3][5] == g["leaf_5"]


def test_golden_insert_single_and_repeated():
    g = GOLD["insert_single"]
    lv = oracle.trie_levels(np.array(g["keys"]), g["p"])
    path = [lv[l][5 >> (g["p"] - l)] for l in range(g["p"] + 1)]
    assert path == [g["path_counters"]] * (g["p"] + 1)
    g = GOLD["insert_zero_repeated"]
    lv = oracle.trie_levels(np.full(g["repeat"], g["key"]), g["p"])
    assert [lv[l][0] for l in range(g["p"] + 1)] == [g["leftmost_path"]] * (g["p"] + 1)


def test_golden_get_item_get_index():
    g = GOLD["get_item_1_5_5"]
    lv = oracle.trie_levels(np.array(g["keys"]), g["p"])
    assert [oracle.get_item(lv, g["p"], r) for r in g["ranks"]] == g["items"]
    g2 = GOLD["get_index_1_5_5"]
    assert [oracle.get_index(lv, g2["p"], v) for v in g2["values"]] == g2["indices"]
    g3 = GOLD["get_item_empty"]
    lv0 = oracle.trie_levels(np.array([], dtype=np.uint64), g3["p"])
    assert oracle.get_item(lv0, g3["p"], g3["rank"], g3["default"]) == g3["item"]
    g4 = GOLD["get_item_singleton"]
    assert oracle.get_item(oracle.trie_levels(np.array(g4["keys"]), g4["p"]), g4["p"], g4["rank"]) == g4["item"]


def test_golden_counter_width():
    for c in GOLD["counter_width"]["cases"]:
        assert oracle.counter_width(c["level"], c["capacity"], c["min"]) == c["width"]


def test_golden_decompose_bit_reverse():
    g = GOLD["decompose"]
    assert g["key"] == int(g["key_binary"], 2)
    assert oracle.decompose(g["key"], g["p"], g["l_n"], g["l_b"]) == (g["bin"], g["offset"], g["trailing"])
    g = GOLD["bit_reverse"]
    assert oracle.bit_reverse(g["x"], g["width"]) == g["reversed"]


def test_golden_alg5_pipeline_3_0_2_2():
    g = GOLD["build_bins_3_0_2_2"]
    C, E = oracle.build_bins(np.array(g["keys"]), g["p"], g["l_n"], g["l_b"])
    assert C.tolist() == g["C"]
    assert E[int(C[0]):].tolist() == g["bin1_offsets_arrival_order"]  # t = 0: entry = offset
    gs = GOLD["sort_bin_1_0_0"]
    assert oracle.sort_bin(np.array(gs["entries"])).tolist() == gs["I"]
    I = np.concatenate([oracle.sort_bin(E[:int(C[0])]), oracle.sort_bin(E[int(C[0]):])])
    K = oracle.reconstruct_all(E, I, C, g["p"], g["l_n"], g["l_b"])
    assert K.tolist() == GOLD["reconstruct_3_0_2_2"]["K"]
    go = GOLD["oracle_sort"]
    assert oracle.sort_u16(np.array(go["keys"], dtype=np.uint16)).tolist() == go["sorted"]
    gl = GOLD["lsb_radix"]
    assert oracle.sort_keys_u64(np.array(gl["keys"], dtype=np.uint64), gl["p"]).tolist() == gl["sorted"]


def test_golden_unit_throughput_and_beff():
    for c in GOLD["unit_throughput"]["cases"]:
        got = metrics.unit_throughput(c["n"], c["t"], c["n_c"])
        assert f"{got:.4g}" == f"{c['keys_per_s']:.4g}", (c["who"], got)
    g = GOLD["bandwidth_efficiency"]
    assert metrics.bandwidth_efficiency(g["useful"], g["total"]) == g["b_eff"]


# ------------------------------------------------------------- brute force on tiny inputs
def test_exhaustive_2bit_sequences_len_le_5():
    for L in range(0, 6):
        for seq in itertools.product(range(4), repeat=L):
            a = np.array(seq, dtype=np.uint16)
            assert oracle.sort_u16(a).tolist() == sorted(seq)
            if L:
                for l_b in (0, 1, 2):
                    assert oracle.alg5_sort(a.astype(np.uint64), 2, l_b)[0].tolist() == sorted(seq)


def test_exhaustive_1bit_sequences_len_8_pairs_stable():
    for seq in itertools.product(range(2), repeat=8):
        k = np.array(seq, dtype=np.uint64)
        v = np.arange(8, dtype=np.uint32)
        ko, vo = oracle.sort_pairs_u64_u32(k, v, 1)
        want = sorted(range(8), key=lambda i: (seq[i], i))  # stable by definition
        assert vo.tolist() == want and ko.tolist() == [seq[i] for i in want]


# ------------------------------------------------------------- library routines / definitions
SIZES = [0, 1, 2, 31, 32, 33, 65535, 65536, 65537, (1 << 20) + 7]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", ["uniform", "zipf", "gauss", "const"])
def test_sort_u16_matches_numpy(n, dist):
    k = datagen.gen_u16(dist, n, seed=n + 1)
    np.testing.assert_array_equal(oracle.sort_u16(k), np.sort(k, kind="stable"))


@pytest.mark.parametrize("threads", [1, 2, 3, 7, 16])
@pytest.mark.parametrize("n", [0, 1, 5, 65_537, 1_000_003])
def test_sort_u16_mt_equals_single_thread(n, threads):
    """The timing-only multi-threaded oracle (PAPER.md:86-92 local -> global
    scheme) is pinned to the single-threaded oracle, every distribution."""
    for dist in ("uniform", "zipf", "sortedswap", "const"):
        k = datagen.gen_u16(dist, n, seed=n + threads)
        np.testing.assert_array_equal(oracle.sort_u16_mt(k, threads), oracle.sort_u16(k))


def test_histogram_matches_bincount_and_scan_matches_cumsum():
    k = datagen.gen_u16("zipf", 1_000_003, seed=3)
    C = oracle.histogram_u16(k)
    np.testing.assert_array_equal(C, np.bincount(k, minlength=65536).astype(np.uint64))
    P = oracle.exclusive_scan(C)
    assert P[0] == 0 and P[-1] == k.size
    np.testing.assert_array_equal(P[1:], np.cumsum(C, dtype=np.uint64))
    # GetIndex(v) = #keys < v (Alg. 3): the lower bound in the sorted array
    s = np.sort(k)
    vs = np.array([0, 1, 100, 32768, 65535], dtype=np.uint16)
    np.testing.assert_array_equal(P[vs.astype(np.int64)], np.searchsorted(s, vs, side="left"))


def test_reconstruct_ranges_are_slices():
    k = datagen.gen_u16("gauss", 200_000, seed=1)
    C = oracle.histogram_u16(k)
    full = oracle.reconstruct_counts_u16(C)
    np.testing.assert_array_equal(full, np.sort(k))
    for b, e in [(0, 0), (0, 1), (199_999, 200_000), (1234, 99_999), (5, 5)]:
        np.testing.assert_array_equal(oracle.reconstruct_counts_u16(C, b, e), full[b:e])


@pytest.mark.parametrize("p", [8, 16])
@pytest.mark.parametrize("dist", ["uniform", "const"])
def test_trie_conservation_sibling_sum_and_queries(p, dist):
    rng = np.random.default_rng(p)
    k = rng.integers(0, 1 << p, size=10_000, dtype=np.uint64) if dist == "uniform" else \
        np.full(10_000, (1 << p) - 3, dtype=np.uint64)
    lv = oracle.trie_levels(k, p)
    for l in range(p + 1):
        assert int(lv[l].sum()) == k.size  # CONSERVATION
    for l in range(p):
        np.testing.assert_array_equal(lv[l], lv[l + 1][0::2] + lv[l + 1][1::2])  # SIBLING SUM
    np.testing.assert_array_equal(lv[p], np.bincount(k.astype(np.int64), minlength=1 << p).astype(np.uint64))
    s = np.sort(k)
    for r in rng.integers(0, k.size, size=100):
        assert oracle.get_item(lv, p, int(r)) == int(s[r])  # ORACLE EQUIVALENCE
    assert oracle.get_item(lv, p, k.size, default=12345) == 12345
    for v in rng.integers(0, 1 << p, size=100):
        assert oracle.get_index(lv, p, int(v)) == int(np.searchsorted(s, v, side="left"))


@pytest.mark.parametrize("p", [8, 16, 32, 64])
@pytest.mark.parametrize("l_b", [0, 1, 4, 8])
@pytest.mark.parametrize("n", [1, 2, 3, 1000, 65537])
def test_alg5_general_matches_numpy(p, l_b, n):
    rng = np.random.default_rng(p * 1000 + l_b * 10 + n)
    hi = np.iinfo(np.uint64).max if p == 64 else (1 << p) - 1
    k = rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)
    out, C = oracle.alg5_sort(k, p, l_b)
    np.testing.assert_array_equal(out, np.sort(k))
    assert int(C.sum()) == n
    # n_bins = 2^(l_n - l_b) (Alg. 5) with l_n = min(p, ceil(log2 n)) from int.bit_length
    l_n = min(p, (n - 1).bit_length())
    assert C.size == 1 << (l_n - min(l_b, l_n))


@pytest.mark.parametrize("p", [1, 8, 16, 64])
@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 2**16 - 1, 2**16, 2**16 + 1, 2**33 + 7])
def test_trie_depth_is_min_p_ceil_log2_n(n, p):
    """l_n = min(p, ceil(log2 n)) (§III.B.1): the expected value comes
    from Python's exact integer bit_length (ceil(log2 n) = (n - 1).bit_length() for n >= 1; 0 for
    n <= 1, a one-key trie has no levels), so a floor/ceil or power-of-two slip fails here."""
    want = min(p, (n - 1).bit_length()) if n >= 1 else 0
    assert oracle.trie_depth(n, p) == want


def test_decompose_round_trip():
    rng = np.random.default_rng(0)
    for key in rng.integers(0, 1 << 32, size=1000, dtype=np.uint64):
        for (p, l_n, l_b) in [(32, 20, 8), (32, 32, 0), (32, 10, 10), (40, 16, 3)]:
            b, o, t = oracle.decompose(int(key), p, l_n, l_b)
            tb = p - l_n
            assert (b << (l_b + tb)) | (o << tb) | t == int(key)  # SPEC.md:182 recomposition


def test_bit_reverse_involution_exhaustive():
    for w in range(1, 17):  # SPEC.md:233, acceptance criterion 9
        xs = range(1 << w) if w <= 12 else range(0, 1 << w, 97)
        for x in xs:
            assert oracle.bit_reverse(oracle.bit_reverse(x, w), w) == x
    assert all(oracle.bit_reverse(x, 1) == x for x in (0, 1))


@pytest.mark.parametrize("key_bits", [1, 8, 16, 17, 33, 64])
def test_sort_pairs_matches_stable_argsort(key_bits):
    n = 200_003
    k = datagen.gen_u64(n, seed=key_bits, key_bits=key_bits)
    v = datagen.iota_u32(n)
    ko, vo = oracle.sort_pairs_u64_u32(k, v, key_bits)
    idx = np.argsort(k, kind="stable")
    np.testing.assert_array_equal(ko, k[idx])
    np.testing.assert_array_equal(vo, idx.astype(np.uint32))
    assert oracle.check_pairs_index(k, ko, vo) == 0


def test_sort_keys_u32_and_u64_match_numpy():
    k = datagen.gen_u32(300_001, seed=2)
    np.testing.assert_array_equal(oracle.sort_keys_u32(k), np.sort(k))
    k = datagen.gen_u64(300_001, seed=2)
    np.testing.assert_array_equal(oracle.sort_keys_u64(k), np.sort(k))


def test_checkers_detect_corruption():
    n = 10_000
    k = datagen.gen_u64(n, seed=5) & np.uint64(0xFF)  # many duplicates
    v = datagen.iota_u32(n)
    ko, vo = oracle.sort_pairs_u64_u32(k, v)
    assert oracle.check_pairs_index(k, ko, vo) == 0
    j = int(np.nonzero(ko[1:] == ko[:-1])[0][0])  # an adjacent equal pair
    bad = vo.copy(); bad[j], bad[j + 1] = bad[j + 1], bad[j]
    assert oracle.check_pairs_index(k, ko, bad) != 0           # stability violation
    bad = vo.copy(); bad[0] = bad[1]
    assert oracle.check_pairs_index(k, ko, bad) != 0           # not a permutation
    badk = ko.copy(); badk[-1] = 0
    assert oracle.check_pairs_index(k, badk, vo) != 0          # order / gather


def test_checker_gather_clause_alone():
    """A mutation that only the gather clause kout[j] == kin[vout[j]] can catch (oracle.c,
    oracle_check_pairs_index): distinct keys (so no stability constraint applies), kout left sorted,
    and two values swapped (so vout is still a permutation).  A checker without the gather clause
    passes it; the real one must report the first swapped position."""
    n = 4_096
    k = datagen.gen_u64(n, seed=11)
    assert np.unique(k).size == n
    v = datagen.iota_u32(n)
    ko, vo = oracle.sort_pairs_u64_u32(k, v)
    assert oracle.check_pairs_index(k, ko, vo) == 0
    for j, jj in ((0, n - 1), (17, 18), (1000, 3000)):
        bad = vo.copy(); bad[j], bad[jj] = bad[jj], bad[j]
        assert np.all(ko[1:] > ko[:-1])                              # order holds, no ties
        assert np.array_equal(np.sort(bad), v)                       # still a permutation
        assert oracle.check_pairs_index(k, ko, bad) == j + 1         # caught at the first swapped slot
    s = oracle.sort_u16(datagen.gen_u16("uniform", 1000))
    assert oracle.check_nondecreasing_u16(s) == 0
    s[10], s[500] = s[500], s[10]
    assert oracle.check_nondecreasing_u16(s) != 0


# ------------------------------------------------------------- closed forms
def test_closed_forms_const_and_sortedswap():
    n = 1_000_000
    k = datagen.gen_u16("const", n)
    np.testing.assert_array_equal(oracle.sort_u16(k), k)
    C = oracle.histogram_u16(k)
    assert C[0xA5A5] == n and C.sum() == n
    k = datagen.gen_u16("sortedswap", n)
    base = ((np.arange(n, dtype=np.uint64) * 65536) // n).astype(np.uint16)
    np.testing.assert_array_equal(oracle.sort_u16(k), base)
    assert int((k != base).sum()) > 0  # the swaps really happened


# ------------------------------------------------------------- multi-rank partition plan
def _send_counts_bruteforce(shards, G):
    """Tag every key (value, rank, local index), sort lexicographically, cut the
    global order into the equal ranges [floor(dN/G), floor((d+1)N/G)) and count."""
    tags = [(int(v), r, i) for r, s in enumerate(shards) for i, v in enumerate(s)]
    tags.sort()
    N = len(tags)
    bounds = [(d * N) // G for d in range(G + 1)]
    out = np.zeros((G, G), dtype=np.uint64)  # out[g][d]
    for pos, (_, r, _) in enumerate(tags):
        d = max(i for i in range(G) if bounds[i] <= pos)
        out[r][d] += 1
    return out


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_send_counts_bruteforce(G):
    rng = np.random.default_rng(G)
    shards = [rng.integers(0, 16, size=rng.integers(0, 40), dtype=np.uint16) for _ in range(G)]
    C_all = np.stack([np.bincount(s, minlength=16).astype(np.uint64) for s in shards])
    want = _send_counts_bruteforce(shards, G)
    for g in range(G):
        np.testing.assert_array_equal(oracle.send_counts(C_all, g), want[g])


# ------------------------------------------------------------- NEXT-3: tapered bit-packed trie export
def test_golden_trie_pack_hand_example():
    g = GOLD["trie_pack_1_3_3"]
    lv = oracle.trie_levels(np.array(g["keys"]), g["p"])
    w, off, words = oracle.trie_pack(lv, g["p"], g["capacity"], g["min_width"])
    assert w.tolist() == g["widths"]
    assert off.tolist() == g["bit_offsets"]
    assert words.tolist() == g["words"]


def _unpack(words, off, w, p):
    """Independent reader: Python big-integer bit slicing of the packed stream."""
    big = 0
    for i, x in enumerate(words.tolist()):
        big |= int(x) << (64 * i)
    out = []
    for l in range(p + 1):
        out.append(np.array([(big >> (int(off[l]) + i * int(w[l]))) & ((1 << int(w[l])) - 1)
                             for i in range(1 << l)], dtype=np.uint64))
    return out


@pytest.mark.parametrize("dist,n,p", [("uniform", 5000, 10), ("const", 777, 8), ("zipf", 20000, 12)])
def test_trie_pack_roundtrip_and_widths(dist, n, p):
    keys = datagen.gen_u16(dist, n, seed=3).astype(np.uint64) >> np.uint64(16 - p)
    lv = oracle.trie_levels(keys, p)
    w, off, words = oracle.trie_pack(lv, p, n, 2)
    back = _unpack(words, off, w, p)
    for l in range(p + 1):
        np.testing.assert_array_equal(back[l], lv[l])
        need = int(lv[l].max()).bit_length()
        base = oracle.counter_width(l, n, 2)
        # tapered width, promoted by exactly as many +4 steps as the level's largest count requires
        k = 0 if need <= base else -(-(need - base) // 4)
        assert w[l] == min(64, base + 4 * k)
        assert int(off[l + 1]) - int(off[l]) == (1 << l) * int(w[l])
