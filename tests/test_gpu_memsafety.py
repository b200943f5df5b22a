"""Memory-safety and race evidence for the CUDA path without compute-sanitizer
(which is closed on this GPU pool: runs under it have left GPUs needing a reset,
profiles/r02/sanitizer_closed.txt).  Each check is the in-repo analogue of one
sanitizer tool, through the C ABI with buffers the test owns:

* memcheck (writes): every output sits between guard zones of 4 KiB filled with
  0xA5; after the call the guards must be untouched (an out-of-bounds write
  below or above an output -- including the peer buffers of the fused exchange
  -- changes them).  Outputs are also placed at misaligned offsets.
* initcheck (temp reads): the temp buffer is filled with 0x00, 0xFF and random
  bytes before each call; the result must be identical and equal the oracle (a
  kernel that read temp it had not written would see different garbage).
* racecheck / synccheck (nondeterminism): each call runs several times with
  different temp garbage; every output must be bit-identical (a shared-memory
  race, a missing barrier or a lookback that reads a stale status word shows up
  as run-to-run differences at these sizes).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_2605_10390_b200 as fs
from paper_2605_10390_b200 import _lib

pytestmark = pytest.mark.gpu

GUARD = 4096
FILLS = ("zero", "ones", "rand1", "rand2")


class Guarded:
    """A device output of nbytes at byte offset `off` inside guard zones."""

    def __init__(self, nbytes, dev, off=0):
        self.n, self.off = nbytes, off
        self.buf = torch.full((GUARD + off + nbytes + GUARD,), 0xA5, dtype=torch.uint8, device=dev)

    def ptr(self):
        return self.buf.data_ptr() + GUARD + self.off

    def data(self, dtype):
        b = self.buf[GUARD + self.off: GUARD + self.off + self.n].cpu().numpy()
        return b.view(dtype)

    def guards_ok(self):
        lo = self.buf[: GUARD + self.off]
        hi = self.buf[GUARD + self.off + self.n:]
        return bool((lo == 0xA5).all().item()) and bool((hi == 0xA5).all().item())


def temp_filled(nbytes, dev, how, seed=0):
    t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    if how == "zero":
        t.zero_()
    elif how == "ones":
        t.fill_(0xFF)
    else:
        g = torch.Generator(device=dev)
        g.manual_seed(seed + (1 if how == "rand1" else 2))
        t.random_(0, 256, generator=g)
    return t


def stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("n,dist", [(100_003, "zipf"), (262_144, "const"), (3_000_017, "uniform"),
                                    (3_000_017, "sortedswap"), (5_000_011, "const")])
@pytest.mark.parametrize("off", [0, 2, 10])
def test_sort_keys_u16_guards_temp_garbage_determinism(cuda, n, dist, off):
    L = fs.lib()
    k = datagen.gen_u16(dist, n, seed=n)
    kin = torch.from_numpy(k).to(cuda)
    want = oracle.sort_u16(k)
    tb = L.fs_sort_keys_u16_temp_bytes(n)
    for fill in FILLS:
        out = Guarded(2 * n, cuda, off)
        temp = temp_filled(tb, cuda, fill, seed=n)
        _lib.check(L.fs_sort_keys_u16(kin.data_ptr(), out.ptr(), n, 16, temp.data_ptr(), tb, stream()), "sort")
        torch.cuda.synchronize()
        assert out.guards_ok(), fill
        np.testing.assert_array_equal(out.data(np.uint16), want, err_msg=fill)


@pytest.mark.parametrize("n,kind", [(5_000, "lsd_one_cta"), (60_000, "msd_small_bins"), (400_003, "msd_local"),
                                    (200_003, "msd_heavy"), (1_000_003, "lsd_24bit")])
def test_sort_pairs_guards_temp_garbage_determinism(cuda, n, kind):
    L = fs.lib()
    kb = 24 if kind == "lsd_24bit" else 64
    k = datagen.gen_u64(n, seed=11, key_bits=kb)
    if kind == "msd_local":  # bins of ~4K keys
        k = (k & np.uint64((1 << 48) - 1)) | ((k >> np.uint64(48)) % np.uint64(100) << np.uint64(48))
    if kind == "msd_heavy":  # 30,000 keys under one 16-bit prefix: recursion into an oversize bin
        k[:30_000] = (k[:30_000] & np.uint64((1 << 48) - 1)) | np.uint64(0x4D2 << 48)
    v = datagen.iota_u32(n)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, kb)
    kd, vd = torch.from_numpy(k).to(cuda), torch.from_numpy(v).to(cuda)
    tb = L.fs_sort_pairs_u64_u32_temp_bytes(n, kb)
    for fill in FILLS:
        ko, vo = Guarded(8 * n, cuda), Guarded(4 * n, cuda)
        temp = temp_filled(tb, cuda, fill, seed=n)
        _lib.check(L.fs_sort_pairs_u64_u32(kd.data_ptr(), vd.data_ptr(), ko.ptr(), vo.ptr(), n, kb, temp.data_ptr(),
                                           tb, stream()), "sort_pairs")
        torch.cuda.synchronize()
        assert ko.guards_ok() and vo.guards_ok(), fill
        np.testing.assert_array_equal(ko.data(np.uint64), ek, err_msg=fill)
        np.testing.assert_array_equal(vo.data(np.uint32), ev, err_msg=fill)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("n", [7_777, 2_000_003])
def test_sort_keys_wide_guards_temp_garbage(cuda, width, n):
    L = fs.lib()
    if width == 32:
        k = datagen.gen_u32(n, seed=n)
        want, tb, fn, dt = oracle.sort_keys_u32(k), L.fs_sort_keys_u32_temp_bytes(n, 0), L.fs_sort_keys_u32, np.uint32
    else:
        k = datagen.gen_u64(n, seed=n)
        want, tb, fn, dt = oracle.sort_keys_u64(k), L.fs_sort_keys_u64_temp_bytes(n, 0), L.fs_sort_keys_u64, np.uint64
    kd = torch.from_numpy(k).to(cuda)
    for fill in FILLS:
        out = Guarded(k.nbytes, cuda)
        temp = temp_filled(tb, cuda, fill, seed=n)
        _lib.check(fn(kd.data_ptr(), out.ptr(), n, 0, temp.data_ptr(), tb, stream()), "sort_keys_wide")
        torch.cuda.synchronize()
        assert out.guards_ok(), fill
        np.testing.assert_array_equal(out.data(dt), want, err_msg=fill)


def test_phase_api_guards(cuda):
    """fs_histogram_u16 (accumulate), fs_exclusive_scan_u64, fs_expand_u16 and the
    two-level fs_histogram_prefix_u16 / fs_expand_prefix_u16, outputs guarded."""
    L = fs.lib()
    n = 1_234_567
    k = datagen.gen_u16("gauss", n, seed=3)
    kd = torch.from_numpy(k).to(cuda)
    C = oracle.histogram_u16(k)
    for fill in FILLS:
        hist = Guarded(8 * 65536, cuda)
        tb = L.fs_histogram_u16_temp_bytes(n)
        temp = temp_filled(tb, cuda, fill)
        _lib.check(L.fs_histogram_u16(kd.data_ptr(), n, 16, hist.ptr(), 0, temp.data_ptr(), tb, stream()), "hist")
        _lib.check(L.fs_histogram_u16(kd.data_ptr(), n, 16, hist.ptr(), 1, temp.data_ptr(), tb, stream()), "hist+")
        pre = Guarded(8 * 65537, cuda)
        sb = L.fs_exclusive_scan_u64_temp_bytes(65536)
        stemp = temp_filled(sb, cuda, fill)
        _lib.check(L.fs_exclusive_scan_u64(hist.ptr(), pre.ptr(), 65536, stemp.data_ptr(), sb, stream()), "scan")
        ex = Guarded(2 * 500_000, cuda, 6)
        _lib.check(L.fs_expand_u16(pre.ptr(), 65536, 300_000, 800_000, ex.ptr(), stream()), "expand")
        p2 = Guarded(8 * (65536 + 128), cuda)
        _lib.check(L.fs_histogram_prefix_u16(kd.data_ptr(), n, p2.ptr(), temp.data_ptr(), tb, stream()), "hist_prefix")
        ex2 = Guarded(2 * 700_000, cuda, 2)
        _lib.check(L.fs_expand_prefix_u16(p2.ptr(), 100_000, 800_000, ex2.ptr(), stream()), "expand_prefix")
        torch.cuda.synchronize()
        for g in (hist, pre, ex, p2, ex2):
            assert g.guards_ok(), fill
        np.testing.assert_array_equal(hist.data(np.uint64), 2 * C)
        np.testing.assert_array_equal(pre.data(np.uint64), oracle.exclusive_scan(2 * C))
        np.testing.assert_array_equal(ex.data(np.uint16), oracle.reconstruct_counts_u16(2 * C, 300_000, 800_000))
        np.testing.assert_array_equal(ex2.data(np.uint16), oracle.reconstruct_counts_u16(C, 100_000, 800_000))


@pytest.mark.parametrize("dist", ["uniform", "zipf", "const"])
def test_expand_to_peers_guards(cuda, dist):
    """The fused exchange writes only inside the owners' ranges (G = 3 virtual
    ranks, every destination guarded and misaligned), whatever temp holds."""
    import ctypes
    L = fs.lib()
    n = 3_000_001
    keys = datagen.gen_u16(dist, n, seed=9)
    cuts = [0, 700_000, 2_100_000, n]
    G = 3
    H = np.stack([oracle.histogram_u16(keys[cuts[r]:cuts[r + 1]]) for r in range(G)])
    hd = torch.from_numpy(H.astype(np.int64)).to(cuda)
    bounds = [(n * d) // G for d in range(G + 1)]
    want = oracle.sort_u16(keys)
    tb = L.fs_expand_to_peers_u16_temp_bytes(65536, G)
    for fill in FILLS:
        dest = [Guarded(2 * (bounds[d + 1] - bounds[d]), cuda, 2 * d) for d in range(G)]
        ptrs = (ctypes.c_void_p * G)(*[g.ptr() for g in dest])
        for g in range(G):
            temp = temp_filled(tb, cuda, fill, seed=g)
            _lib.check(L.fs_expand_to_peers_u16(hd.data_ptr(), G, g, 65536, ptrs, temp.data_ptr(), tb, stream()),
                       "expand_to_peers")
            torch.cuda.synchronize()
        for g in dest:
            assert g.guards_ok(), fill
        got = np.concatenate([g.data(np.uint16) for g in dest])
        np.testing.assert_array_equal(got, want, err_msg=fill)


def test_repeated_sorts_bit_identical(cuda):
    """20 back-to-back sorts of one input on one stream with one temp buffer, and
    10 on two streams at once with their own temps: all outputs identical."""
    n = 1 << 24
    k = torch.empty(n, dtype=torch.uint16, device=cuda)
    datagen.gen_u16_device(k.data_ptr(), "zipf", n, seed=4, stream=stream())
    ref = fs.sort_keys(k)
    outs = [torch.empty_like(k) for _ in range(20)]
    for o in outs:
        fs.sort_keys(k, out=o)
    s2 = torch.cuda.Stream()
    outs2 = []
    with torch.cuda.stream(s2):
        for _ in range(10):
            outs2.append(fs.sort_keys(k))
    torch.cuda.synchronize()
    for o in outs + outs2:
        assert torch.equal(o, ref)
    kp = torch.empty(1 << 22, dtype=torch.uint64, device=cuda)
    datagen.gen_u64_device(kp.data_ptr(), 1 << 22, seed=5, stream=stream())
    vp = torch.empty(1 << 22, dtype=torch.uint32, device=cuda)
    datagen.iota_u32_device(vp.data_ptr(), 1 << 22, stream=stream())
    rk, rv = fs.sort_pairs(kp, vp)
    for _ in range(8):
        ok, ov = fs.sort_pairs(kp, vp)
        assert torch.equal(ok, rk) and torch.equal(ov, rv)


@pytest.mark.parametrize("kind", ["uniform", "ties"])
def test_pair_exchange_guards(cuda, kind):
    """The fused pair exchange (fs_pair_classes_u64 + fs_pair_scatter_u64_u32) writes
    only inside every owner's share (G = 3 virtual ranks, each destination guarded
    and misaligned), whatever its temp holds; the owners' buffers hold exactly the
    pairs the class-order cuts assign them."""
    import ctypes
    L = fs.lib()
    n, G = 200_003, 3
    k = datagen.gen_u64(n, seed=17)
    if kind == "ties":
        k = k & np.uint64(3)
    v = datagen.iota_u32(n)
    order = np.argsort(k, kind="stable")
    K = [int(k[order[(n * d) // G]]) for d in range(1, G)]
    Kd = torch.from_numpy(np.array(K, dtype=np.uint64).view(np.int64)).to(cuda)
    kd, vd = torch.from_numpy(k).to(cuda), torch.from_numpy(v).to(cuda)
    tb = L.fs_pair_exchange_temp_bytes(n, G)
    # classes and cuts by definition (one rank: ties split at the boundary positions)
    d_ = np.searchsorted(np.array(K, dtype=np.uint64), k, side="left")
    tie = np.zeros(n, dtype=bool)
    inside = d_ < len(K)
    tie[inside] = np.array(K, dtype=np.uint64)[d_[inside]] == k[inside]
    cls = 2 * d_ + tie
    cnt = np.bincount(cls, minlength=2 * G - 1)
    start = np.concatenate([[0], np.cumsum(cnt)])
    first = [next(i for i in range(G - 1) if K[i] == K[j]) for j in range(G - 1)]
    cuts = [0]
    for j in range(G - 1):
        below = int((k < np.uint64(K[j])).sum())
        cuts.append(int(start[2 * first[j] + 1]) + ((n * (j + 1)) // G - below))
    cuts.append(n)
    want = np.argsort(cls, kind="stable")
    for fill in FILLS:
        temp = temp_filled(tb, cuda, fill, seed=3)
        tot = torch.empty(2 * G - 1, dtype=torch.int64, device=cuda)
        _lib.check(L.fs_pair_classes_u64(kd.data_ptr(), n, Kd.data_ptr(), G, tot.data_ptr(), temp.data_ptr(), tb,
                                         stream()), "classes")
        np.testing.assert_array_equal(tot.cpu().numpy(), cnt)
        dk = [Guarded(8 * (cuts[d + 1] - cuts[d]), cuda, 8 * d) for d in range(G)]
        dv = [Guarded(4 * (cuts[d + 1] - cuts[d]), cuda, 4 * d) for d in range(G)]
        c_ = (ctypes.c_uint64 * (G + 1))(*cuts)
        b_ = (ctypes.c_uint64 * G)(*([0] * G))
        pk = (ctypes.c_void_p * G)(*[g.ptr() for g in dk])
        pv = (ctypes.c_void_p * G)(*[g.ptr() for g in dv])
        _lib.check(L.fs_pair_scatter_u64_u32(kd.data_ptr(), vd.data_ptr(), n, Kd.data_ptr(), G, c_, b_, pk, pv,
                                             temp.data_ptr(), tb, stream()), "scatter")
        torch.cuda.synchronize()
        for g in dk + dv:
            assert g.guards_ok(), fill
        for d in range(G):
            sel = want[cuts[d]:cuts[d + 1]]
            np.testing.assert_array_equal(dk[d].data(np.uint64), k[sel], err_msg=fill)
            np.testing.assert_array_equal(dv[d].data(np.uint32), v[sel], err_msg=fill)
