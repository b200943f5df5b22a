"""GPU parity of the u16 hot path (histogram -> scan -> count-expansion) against the
CPU oracle, through the C ABI (via the thin binding).  Bar: bit-exact (integer work).

Sizes span several tiles and ragged tails; full-size configs c1-c3 of BASELINE.json
are compared element by element in the launch configuration bench.py times.
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2605_10390_b200 as fs

pytestmark = pytest.mark.gpu


def to_dev(a: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


EDGE_N = [1, 2, 7, 8, 9, 31, 32, 33, 255, 4097, 65535, 65536, 65537, 131071, (1 << 20) + 7, 3_000_001]


@pytest.mark.parametrize("n", EDGE_N)
def test_sort_u16_uniform_edges(cuda, n):
    keys = datagen.gen_u16("uniform", n, seed=n)
    out = fs.sort_keys(to_dev(keys, cuda))
    np.testing.assert_array_equal(to_host(out), oracle.sort_u16(keys))


@pytest.mark.parametrize("dist", ["uniform", "zipf", "gauss", "sortedswap", "const"])
@pytest.mark.parametrize("n", [1000, 65536 * 3 + 5, 1 << 21])
def test_sort_u16_distributions(cuda, dist, n):
    keys = datagen.gen_u16(dist, n, seed=7)
    out = fs.sort_keys(to_dev(keys, cuda))
    np.testing.assert_array_equal(to_host(out), oracle.sort_u16(keys))


@pytest.mark.parametrize("value", [0, 1, 0xA5A5, 65534, 65535])
def test_sort_u16_all_equal(cuda, value):
    n = (1 << 22) + 3  # forces many spills of one hot counter per SM
    keys = np.full(n, value, dtype=np.uint16)
    out = to_host(fs.sort_keys(to_dev(keys, cuda)))
    np.testing.assert_array_equal(out, keys)


@pytest.mark.parametrize("nvals,swap", [(2, 0.01), (16, 0.02), (300, 0.05)])
def test_sort_u16_nearly_sorted_spilling_runs(cuda, nvals, swap):
    """Sorted runs long enough to spill (2^26 keys over a few values, every CTA's
    run counters cross 2^15) with a fraction of random swaps: exercises the
    aggregating path, its queue of mixed vectors (drained 32 at a time and at the
    end of each warp's work) and the spill protocol together."""
    n = (1 << 26) + 5
    rng = np.random.default_rng(nvals)
    vals = np.sort(rng.choice(65536, size=nvals, replace=False)).astype(np.uint16)
    keys = np.repeat(vals, -(-n // nvals))[:n].copy()
    i = rng.integers(0, n, size=int(n * swap))
    j = rng.integers(0, n, size=i.size)
    keys[i], keys[j] = keys[j], keys[i].copy()
    out = to_host(fs.sort_keys(to_dev(keys, cuda)))
    np.testing.assert_array_equal(out, oracle.sort_u16(keys))


def test_sort_u16_two_hot_bins(cuda):
    """Adversarial for the 16-bit packed counters: both halves of one word are hot."""
    n = 1 << 23
    rng = np.random.default_rng(3)
    keys = rng.choice(np.array([4242, 4243], dtype=np.uint16), size=n)
    out = to_host(fs.sort_keys(to_dev(keys, cuda)))
    np.testing.assert_array_equal(out, oracle.sort_u16(keys))


@pytest.mark.parametrize("pattern", ["alternate", "blocks"])
def test_sort_u16_maximal_contention_spill(cuda, pattern):
    """Maximal contention on ONE counter word for a long stretch: 2^31 keys
    (14.5M per CTA, ~220 spill epochs of each half per CTA), every key one of
    the two bins of one 32-bit word (4242 / 4243), so every shared-memory
    atomic of all 1024 threads of every CTA hits the same word and no vector is
    eight equal keys ("alternate"), or runs of 8 equal keys alternate between
    the two halves so every vector is run-aggregated ("blocks").  White-box:
    the kernel's u64 spill array (the first 512 KiB of the temp buffer,
    hist16.cu) must have received the spilled counts of exactly these two bins,
    and the output must be exact.  The spill bound (static_assert in hist16.cu)
    is what keeps the packed u16 halves from wrapping here."""
    from paper_2605_10390_b200 import _lib
    n = 1 << 31
    unit = [4242, 4243] if pattern == "alternate" else [4242] * 8 + [4243] * 8
    keys = torch.tensor(unit, dtype=torch.int16, device=cuda).repeat(n // len(unit)).view(torch.uint16)
    L = fs.lib()
    temp = torch.zeros(L.fs_sort_keys_u16_temp_bytes(n), dtype=torch.uint8, device=cuda)
    out = torch.empty_like(keys)
    _lib.check(L.fs_sort_keys_u16(keys.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(),
                                  torch.cuda.current_stream().cuda_stream), "fs_sort_keys_u16")
    torch.cuda.synchronize()
    half = n // 2
    assert bool((out[:half].view(torch.int16) == 4242).all().item())
    assert bool((out[half:].view(torch.int16) == 4243).all().item())
    spill = temp[: 65536 * 8].view(torch.int64)
    nz = torch.nonzero(spill).flatten().cpu().tolist()
    assert set(nz) == {4242, 4243}
    grid = min(148, torch.cuda.get_device_properties(cuda).multi_processor_count)
    for b in (4242, 4243):  # all but < 2^15 + 49,407 per CTA went through the spill
        assert int(spill[b].item()) >= half - grid * 65536


@pytest.mark.parametrize("n", [1, 9, 4095, 65536, 100_003, (1 << 18) - 1, 1 << 18, (1 << 18) + 1])
@pytest.mark.parametrize("dist", ["uniform", "zipf", "const", "sortedswap"])
def test_sort_u16_one_cluster_path(cuda, n, dist):
    """Sizes up to 2^18 take the one-launch cluster sort (small16.cu); the
    boundary and just above it take the two-kernel path."""
    k = datagen.gen_u16(dist, n, seed=n % 97)
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_u16(k))


@pytest.mark.parametrize("offset", [1, 3, 7])
def test_sort_u16_one_cluster_misaligned_in_place(cuda, offset):
    """The cluster sort with keys and output not 16-byte aligned (scalar loads
    and stores), in place."""
    n = 200_001
    k = datagen.gen_u16("uniform", n + offset, seed=offset)
    d = to_dev(k, cuda)[offset:]
    fs.sort_keys(d, out=d)
    np.testing.assert_array_equal(to_host(d), oracle.sort_u16(k[offset:]))


@pytest.mark.parametrize("hot,frac", [(0xFFFF, 0.5), (0, 0.6), (0x1235, 0.05)])
def test_sort_u16_hot_key(cuda, hot, frac):
    """One key far above the others (a CTA's first spill makes it the warps'
    register-counted hot key): bins at both ends of the table, and a key just
    hot enough to spill in some CTAs only."""
    n = (1 << 24) + 3
    k = datagen.gen_u16("uniform", n, seed=7)
    sel = datagen.gen_u16("uniform", n, seed=8).astype(np.float64) / 65536.0 < frac
    k[sel] = hot
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_u16(k))
    np.testing.assert_array_equal(to_host(fs.histogram_u16(to_dev(k, cuda))).astype(np.uint64), oracle.histogram_u16(k))


def test_sort_u16_hot_key_changes(cuda):
    """The hot key changes halfway (key A, then key B): the CTA keeps its first
    hot key; B's counts go through the shared-memory counters and their spill."""
    n = (1 << 24) + 1
    k = datagen.gen_u16("uniform", n, seed=9)
    sel = datagen.gen_u16("uniform", n, seed=10) < 40000
    half = np.arange(n) < n // 2
    k[sel & half] = 0x0A0A
    k[sel & ~half] = 0xB0B0
    np.testing.assert_array_equal(to_host(fs.sort_keys(to_dev(k, cuda))), oracle.sort_u16(k))


@pytest.mark.parametrize("offset", range(8))
def test_sort_u16_misaligned(cuda, offset):
    """Input and output start at every 2-byte offset of a 16-byte vector."""
    n = 100_003
    keys = datagen.gen_u16("uniform", n + 16, seed=11)
    src = to_dev(keys, cuda)[offset:offset + n]
    dst_buf = torch.empty(n + 16, dtype=torch.uint16, device=cuda)
    dst = dst_buf[(7 * offset) % 8:(7 * offset) % 8 + n]
    fs.sort_keys(src, out=dst)
    np.testing.assert_array_equal(to_host(dst), oracle.sort_u16(keys[offset:offset + n]))


def test_sort_u16_in_place(cuda):
    keys = datagen.gen_u16("zipf", 1 << 20, seed=5)
    t = to_dev(keys, cuda)
    fs.sort_keys(t, out=t)
    np.testing.assert_array_equal(to_host(t), oracle.sort_u16(keys))


def test_sort_u16_empty(cuda):
    t = torch.empty(0, dtype=torch.uint16, device=cuda)
    assert fs.sort_keys(t).numel() == 0


@pytest.mark.parametrize("dist", ["uniform", "zipf", "gauss", "sortedswap", "const"])
def test_histogram_u16(cuda, dist):
    keys = datagen.gen_u16(dist, 5_000_017, seed=2)
    h = to_host(fs.histogram_u16(to_dev(keys, cuda))).astype(np.uint64)
    np.testing.assert_array_equal(h, oracle.histogram_u16(keys))


def test_histogram_u16_accumulate_and_key_bits(cuda):
    a = datagen.gen_u16("uniform", 300_000, seed=1, key_bits=12)
    b = datagen.gen_u16("uniform", 200_001, seed=2, key_bits=12)
    h = fs.histogram_u16(to_dev(a, cuda), key_bits=12)
    fs.histogram_u16(to_dev(b, cuda), key_bits=12, hist=h, accumulate=True)
    want = oracle.histogram_u16(np.concatenate([a, b]))[:4096]
    np.testing.assert_array_equal(to_host(h).astype(np.uint64), want)
    # n = 0 with accumulate = 0 zeroes the histogram
    fs.histogram_u16(torch.empty(0, dtype=torch.uint16, device=cuda), key_bits=12, hist=h, accumulate=False)
    assert int(h.abs().sum()) == 0


@pytest.mark.parametrize("nbins", [1, 2, 255, 256, 257, 4096, 65536, 65536 * 7 + 3])
def test_exclusive_scan(cuda, nbins):
    rng = np.random.default_rng(nbins)
    C = rng.integers(0, 1 << 20, size=nbins, dtype=np.uint64)
    if nbins > 3:
        C[rng.integers(0, nbins, size=nbins // 3)] = 0
    P = to_host(fs.exclusive_scan(to_dev(C.astype(np.int64), cuda))).astype(np.uint64)
    np.testing.assert_array_equal(P, oracle.exclusive_scan(C))


@pytest.mark.parametrize("dist", ["uniform", "const", "zipf"])
def test_expand_ranges(cuda, dist):
    keys = datagen.gen_u16(dist, 777_777, seed=4)
    C = oracle.histogram_u16(keys)
    P = oracle.exclusive_scan(C)
    Pd = to_dev(P.astype(np.int64), cuda)
    full = oracle.reconstruct_counts_u16(C)
    n = keys.size
    for (b, e) in [(0, n), (0, 1), (n - 1, n), (12345, 23456), (1, 9), (n // 3, 2 * n // 3), (5, 5)]:
        out = to_host(fs.expand_u16(Pd, b, e))
        np.testing.assert_array_equal(out, full[b:e])


def test_expand_sparse_bins(cuda):
    """Tiles spanning more bins than the staged slice (the L2 search fallback)."""
    keys = np.concatenate([np.arange(0, 65536, 1, dtype=np.uint16),
                           np.full(50_000, 7, dtype=np.uint16), np.array([65535] * 10, dtype=np.uint16)])
    out = to_host(fs.sort_keys(to_dev(keys, cuda)))
    np.testing.assert_array_equal(out, oracle.sort_u16(keys))


# ------------------------------------------------------------------ full-size configs
@pytest.mark.parametrize("cfg,dist,n", [
    ("c1", "uniform", 1 << 20),
    ("c2", "uniform", 1 << 28),
    ("c3a", "zipf", 1 << 28),
    ("c3b", "gauss", 1 << 28),
    ("c3c", "sortedswap", 1 << 28),
    ("c3d", "const", 1 << 28),
])
def test_full_size_configs(cuda, cfg, dist, n):
    """BASELINE.json configs c1-c3 at full size, compared element by element."""
    if dist in ("uniform", "zipf", "gauss", "const"):
        t = torch.empty(n, dtype=torch.uint16, device=cuda)
        datagen.gen_u16_device(t.data_ptr(), dist, n, seed=0, stream=torch.cuda.current_stream().cuda_stream)
        keys = to_host(t)
    else:
        keys = datagen.gen_u16(dist, n, seed=0)
        t = to_dev(keys, cuda)
    out = to_host(fs.sort_keys(t))
    want = oracle.sort_u16(keys)
    np.testing.assert_array_equal(out, want)
    if dist == "sortedswap":  # closed form: the sorted output is the pre-swap base array
        base = ((np.arange(n, dtype=np.uint64) * 65536) // n).astype(np.uint16)
        np.testing.assert_array_equal(out, base)


def test_device_datagen_matches_host(cuda):
    for dist in ["uniform", "zipf", "gauss", "const"]:
        n = 1_000_003
        t = torch.empty(n, dtype=torch.uint16, device=cuda)
        datagen.gen_u16_device(t.data_ptr(), dist, n, seed=9, i0=12345, stream=torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(to_host(t), datagen.gen_u16(dist, n, seed=9, i0=12345, n_total=n + 12345))


def test_host_streaming_sort(cuda):
    n = (1 << 22) + 5
    keys = datagen.gen_u16("gauss", n, seed=8)
    src = torch.from_numpy(keys).pin_memory()
    out = fs.sort_keys_u16_host(src, batch=1 << 20)
    np.testing.assert_array_equal(out.numpy(), oracle.sort_u16(keys))
    out2 = fs.sort_keys_u16_host(torch.from_numpy(keys), batch=0)  # pageable, default batch
    np.testing.assert_array_equal(out2.numpy(), oracle.sort_u16(keys))


def test_host_streaming_sort_two_streams(cuda):
    """Host-buffer sorts issued on two streams with their own work buffers
    overlap (one call's copy-out with the other's copy-in, on the library's
    separate H2D / D2H copy streams); a third call reuses stream A's work buffer
    in stream order.  Every output must be the oracle's."""
    n = (1 << 23) + 3
    ka = datagen.gen_u16("uniform", n, seed=31)
    kb = datagen.gen_u16("zipf", n, seed=32)
    kc = datagen.gen_u16("sortedswap", n, seed=33)
    srcs = [torch.from_numpy(k).pin_memory() for k in (ka, kb, kc)]
    outs = [torch.empty(n, dtype=torch.uint16).pin_memory() for _ in range(3)]
    need = fs.sort_keys_u16_host_work_bytes(n, 1 << 21)
    wa = torch.empty(need, dtype=torch.uint8, device=cuda)
    wb = torch.empty(need, dtype=torch.uint8, device=cuda)
    sa, sb = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    with torch.cuda.stream(sa):
        fs.sort_keys_u16_host(srcs[0], outs[0], batch=1 << 21, work=wa, synchronize=False)
    with torch.cuda.stream(sb):
        fs.sort_keys_u16_host(srcs[1], outs[1], batch=1 << 21, work=wb, synchronize=False)
    with torch.cuda.stream(sa):
        fs.sort_keys_u16_host(srcs[2], outs[2], batch=1 << 21, work=wa, synchronize=False)
    torch.cuda.synchronize(cuda)
    for k, o in zip((ka, kb, kc), outs):
        np.testing.assert_array_equal(o.numpy(), oracle.sort_u16(k))


def test_send_counts_matches_oracle(cuda):
    rng = np.random.default_rng(0)
    for G in [1, 2, 3, 8]:
        hist_all = np.stack([oracle.histogram_u16(datagen.gen_u16("zipf", 10_000 + 37 * r, seed=r))
                             for r in range(G)])
        Hd = to_dev(hist_all.astype(np.int64), cuda)
        for g in range(G):
            got = to_host(fs.send_counts(Hd, g)).astype(np.uint64)
            np.testing.assert_array_equal(got, oracle.send_counts(hist_all, g))
    del rng


def test_c4_full_size_one_gpu(cuda):
    """Config c4 at full size on one GPU (2^34 keys, 32 GB; bench.py's N = 1
    launch configuration): the oracle histogram of the input, streamed to the
    host in chunks, fixes every value's output range; each value's first and
    last position, 2^20 random positions and the non-decreasing order (checked
    on the device, chunked) must agree — together they pin the sorted multiset."""
    n = 1 << 34
    chunk = 1 << 28
    keys = torch.empty(n, dtype=torch.uint16, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    datagen.gen_u16_device(keys.data_ptr(), "uniform", n, seed=0, n_total=n, stream=s)
    out = fs.sort_keys(keys)
    C = np.zeros(65536, dtype=np.uint64)
    for a in range(0, n, chunk):
        C += oracle.histogram_u16(to_host(keys[a:a + chunk]))
    del keys
    P = oracle.exclusive_scan(C)
    nonempty = np.nonzero(C)[0]
    pos = np.concatenate([P[nonempty], P[nonempty + 1] - 1,
                          np.random.default_rng(0).integers(0, n, 1 << 20).astype(np.uint64)])
    want = (np.searchsorted(P, pos, side="right") - 1).astype(np.int64)
    got = out.view(torch.int16)[torch.from_numpy(pos.astype(np.int64)).to(cuda)].to(torch.int64).cpu().numpy() & 0xFFFF
    np.testing.assert_array_equal(got, want)
    for a in range(0, n - 1, chunk):
        seg = out[a:min(a + chunk + 1, n)].view(torch.int16).to(torch.int32) & 0xFFFF
        assert bool((seg[1:] >= seg[:-1]).all().item()), f"order broken in [{a}, {a + chunk}]"
