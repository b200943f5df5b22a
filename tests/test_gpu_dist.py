"""dist.py's default CudaOps path on one GPU (NCCL process group of size 1):
Mode A and Mode B through the library kernels, checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import datagen
import oracle
from paper_2605_10390_b200 import dist as fsdist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group(cuda):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["B", "A", "P"])
@pytest.mark.parametrize("dist_name", ["uniform", "zipf", "const"])
def test_dist_single_rank(cuda, nccl_group, mode, dist_name):
    keys = datagen.gen_u16(dist_name, 1_000_003, seed=1)
    out, (b, e) = fsdist.sort_keys_u16(torch.from_numpy(keys).to(cuda), mode=mode)
    assert (b, e) == (0, keys.size)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.sort_u16(keys))


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("dist_name", ["uniform", "zipf", "const", "sortedswap"])
def test_expand_to_peers_virtual_ranks(cuda, G, dist_name):
    """fs_expand_to_peers_u16 for every rank g of a G-rank job, issued from one
    GPU into G separate buffers (each call only writes; no call waits on
    another): the buffers concatenate to the oracle sort of the whole input."""
    import paper_2605_10390_b200 as fs
    n = 2_000_003
    keys = datagen.gen_u16(dist_name, n, seed=G)
    cuts = [0] + sorted((n * (2 * r + 1)) // (2 * G) for r in range(1, G)) + [n]  # uneven shards
    hist_all = torch.stack([fs.histogram_u16(torch.from_numpy(keys[cuts[r]:cuts[r + 1]].copy()).to(cuda))
                            for r in range(G)])
    bounds = [(n * d) // G for d in range(G + 1)]
    bufs = [torch.full((bounds[d + 1] - bounds[d],), 0xFFFF, dtype=torch.uint16, device=cuda) for d in range(G)]
    for g in range(G):
        fs.expand_to_peers_u16(hist_all, g, bufs)
    torch.cuda.synchronize()
    got = np.concatenate([b.cpu().numpy() for b in bufs])
    np.testing.assert_array_equal(got, oracle.sort_u16(keys))


@pytest.mark.parametrize("n", [0, 1, 1000, 1_000_003])
def test_bound_u64_matches_searchsorted(cuda, n):
    """fs_bound_u64 (splitter rank counts) = #keys < q / <= q, checked against
    numpy.searchsorted on the same ascending array (duplicates, extremes)."""
    import paper_2605_10390_b200 as fs
    k = np.sort(datagen.gen_u64(n, seed=3) & np.uint64(0xFFFF0000000000FF)) if n else np.zeros(0, np.uint64)
    q = np.concatenate([datagen.gen_u64(500, seed=4), k[:: max(1, n // 100)][:200],
                        np.array([0, 2**64 - 1], dtype=np.uint64)]).astype(np.uint64)
    kd = torch.from_numpy(k).to(cuda)
    qd = torch.from_numpy(q).to(cuda)
    for upper, side in ((False, "left"), (True, "right")):
        got = fs.bound_u64(kd, qd, upper).cpu().numpy()
        np.testing.assert_array_equal(got, np.searchsorted(k, q, side=side).astype(np.int64))


@pytest.mark.parametrize("mode", ["A", "P"])
def test_dist_pairs_single_rank(cuda, nccl_group, mode):
    k = datagen.gen_u64(500_001, seed=5) & np.uint64(0xFF)
    v = datagen.iota_u32(500_001)
    (ko, vo), (b, e) = fsdist.sort_pairs_u64_u32(torch.from_numpy(k).to(cuda), torch.from_numpy(v).to(cuda),
                                                 mode=mode)
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    assert (b, e) == (0, k.size)
    np.testing.assert_array_equal(ko.cpu().numpy(), ek)
    np.testing.assert_array_equal(vo.cpu().numpy(), ev)


@pytest.mark.parametrize("dist_name", ["uniform", "zipf", "const"])
def test_two_level_prefix_sum_over_ranks(cuda, dist_name):
    """fs_histogram_prefix_u16 of shards summed element-wise (what the all-reduce
    does) and expanded per output range = the oracle sort of the union."""
    import paper_2605_10390_b200 as fs
    keys = datagen.gen_u16(dist_name, 3_000_017, seed=7)
    cuts = [0, 700_001, 2_100_000, keys.size]
    p2 = sum(fs.histogram_prefix_u16(torch.from_numpy(keys[a:b].copy()).to(cuda)) for a, b in zip(cuts, cuts[1:]))
    want = oracle.sort_u16(keys)
    for a, b in [(0, keys.size), (0, 1), (12345, 1_234_567), (keys.size - 9, keys.size)]:
        np.testing.assert_array_equal(fs.expand_prefix_u16(p2, a, b).cpu().numpy(), want[a:b])


def _virtual_pair_sort(cuda, k, v, G, cuts_in, key_bits=64):
    """The distributed pair sort of dist.sort_pairs_u64_u32 mode "P" for G virtual
    ranks on one GPU: the collectives become host sums, every other step is the
    library's (fs_histogram16_u64, fs_select_bins_u64, fs_sort_keys_u64,
    fs_digit_counts_sorted_u64, fs_pair_classes_u64, fs_pair_scatter_u64_u32 into
    G separate owner buffers, fs_sort_pairs_u64_u32 per owner)."""
    import paper_2605_10390_b200 as fs
    from paper_2605_10390_b200 import dist as fsd
    N = k.size
    shards = [(torch.from_numpy(k[cuts_in[r]:cuts_in[r + 1]].copy()).to(cuda),
               torch.from_numpy(v[cuts_in[r]:cuts_in[r + 1]].copy()).to(cuda)) for r in range(G)]
    nr = [cuts_in[r + 1] - cuts_in[r] for r in range(G)]
    levels = fsd._levels(key_bits)
    bounds = [(N * d) // G for d in range(1, G)]
    (s1, w1) = levels[0]
    h1 = [fs.histogram16_u64(sk, s1, w1) for sk, _ in shards]
    K, L = fsd.splitter_level1(sum(h.cpu().numpy() for h in h1), bounds, s1)
    bins = sorted({x >> s1 for x in K})
    cands = []
    for (sk, _), h in zip(shards, h1):
        cap = int(h[torch.tensor(bins, device=cuda)].sum().item())
        c = fs.select_bins_u64(sk, s1, w1, bins, cap)
        cands.append(fs.sort_keys(c) if c.numel() else c)
    for shift, width in levels[1:]:
        Hl = sum(fs.digit_counts_sorted_u64(c, K, shift, width).cpu().numpy() for c in cands)
        fsd.splitter_refine(Hl, bounds, K, L, shift)
    exs = [fs.PairExchange(sk, sv, K, G) for sk, sv in shards]
    T_all = np.array([ex.classes() for ex in exs], dtype=np.int64)
    cuts_all = fsd.pair_cuts(T_all, K, L, bounds, nr)
    owners = [(N * d) // G for d in range(G + 1)]
    dk = [torch.empty(owners[d + 1] - owners[d], dtype=torch.uint64, device=cuda) for d in range(G)]
    dv = [torch.empty(owners[d + 1] - owners[d], dtype=torch.uint32, device=cuda) for d in range(G)]
    for r, ex in enumerate(exs):
        bases = [sum(cuts_all[q][d + 1] - cuts_all[q][d] for q in range(r)) for d in range(G)]
        ex.scatter(cuts_all[r], bases, dk, dv)
    torch.cuda.synchronize()
    outk, outv = [], []
    for d in range(G):
        if dk[d].numel():
            a, b = fs.sort_pairs(dk[d], dv[d])
            outk.append(a.cpu().numpy())
            outv.append(b.cpu().numpy())
    return np.concatenate(outk), np.concatenate(outv), K


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("kind", ["uniform", "ties8", "const", "hi16", "ties3"])
def test_fused_pair_exchange_virtual_ranks(cuda, G, kind):
    """NEXT-2 for pairs on one GPU: exact splitters from the CUDA histogram levels,
    the classes + peer-store scatter into G owner buffers, one stable sort per
    owner; the owners' outputs concatenate to the oracle's stable sort (values =
    arrival indices, so stability is checked)."""
    n = 300_007
    k = datagen.gen_u64(n, seed=G)
    if kind == "ties8":
        k = k & np.uint64(7)
    elif kind == "const":
        k = np.full(n, 0x0123456789ABCDEF, dtype=np.uint64)
    elif kind == "hi16":
        k = (k & np.uint64((1 << 48) - 1)) | np.uint64(0xBEEF << 48)
    elif kind == "ties3":
        k = (k % np.uint64(3)) << np.uint64(62)
    v = datagen.iota_u32(n)
    cuts = [0] + sorted((n * (2 * r + 1)) // (2 * G) for r in range(1, G)) + [n]  # uneven shards
    gk, gv, K = _virtual_pair_sort(cuda, k, v, G, cuts)
    ek, ev = oracle.sort_pairs_u64_u32(k, v)
    np.testing.assert_array_equal(gk, ek)
    np.testing.assert_array_equal(gv, ev)
    # the splitters are exactly the keys at the rank boundaries
    assert K == [int(ek[(n * d) // G]) for d in range(1, G)]


# ---------------------------------------------------------------- mode "N": NVLS multicast
@pytest.fixture(scope="module")
def mcbuf(cuda, nccl_group):
    from cuda.bindings import driver as cu
    err, d = cu.cuDeviceGet(cuda.index)
    err, mc_ok = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)
    if mc_ok != 1:
        pytest.skip("the device reports no multicast (NVLS) support")
    try:
        b = fsdist.MulticastBuffer(65536 + 128, cuda)
    except RuntimeError as e:
        # The pool's one-GPU boxes report multicast support but the driver refuses to
        # create any multicast object (CUDA_ERROR_INVALID_VALUE for every size, handle
        # type and device count, from C as well: GPU fabric GUID 0, no NVSwitch
        # fabric in the slice; profiles/r02g/nvls_probe.txt).  Any other failure fails.
        if "cuMulticastCreate failed" not in str(e):
            raise
        pytest.skip(f"no NVSwitch multicast fabric on this box: {e}")
    yield b
    b.close()


def _to_raw(dst_ptr, t):
    from cuda.bindings import driver as cu
    torch.cuda.synchronize()
    (err,) = cu.cuMemcpyDtoD(dst_ptr, t.data_ptr(), t.numel() * t.element_size())
    assert err == cu.CUresult.CUDA_SUCCESS, err
    torch.cuda.synchronize()


@pytest.mark.parametrize("count", [1, 1000, 65536 + 128])
def test_allreduce_multicast_single_rank(cuda, mcbuf, count):
    """fs_allreduce_multicast_u64 through the multicast mapping of a one-GPU
    multicast group: every element comes back through multimem.ld_reduce equal
    to what the rank wrote (the sum over one rank), on both halves, over several
    calls (the flag's target grows by G = 1 per call); count = 0 is a pure barrier."""
    import paper_2605_10390_b200 as fs
    gen = torch.Generator().manual_seed(count)
    for call in range(4):
        src = torch.randint(-(1 << 62), 1 << 62, (count,), generator=gen, dtype=torch.int64).to(cuda)
        uc, mc, fmc, fl, target = mcbuf.step()
        _to_raw(uc, src)
        dst = torch.full((count,), -1, dtype=torch.int64, device=cuda)
        _, timed_out = fs.allreduce_multicast_u64(mc, dst, fmc, fl, target)
        torch.cuda.synchronize()
        assert int(timed_out.item()) == 0
        assert torch.equal(dst, src), (count, call)
    uc, mc, fmc, fl, target = mcbuf.step()
    _, timed_out = fs.allreduce_multicast_u64(mc, torch.empty(0, dtype=torch.int64, device=cuda), fmc, fl, target)
    torch.cuda.synchronize()
    assert int(timed_out.item()) == 0
    # a target no rank will reach (a missing peer): the call gives up after its timeout, dst untouched
    uc, mc, fmc, fl, target = mcbuf.step()
    dst = torch.full((count,), -1, dtype=torch.int64, device=cuda)
    _, timed_out = fs.allreduce_multicast_u64(mc, dst, fmc, fl, target + 5, timeout_s=0.05)
    torch.cuda.synchronize()
    assert int(timed_out.item()) == 1 and bool((dst == -1).all())   # (the flag still counts this arrival: G x calls)


@pytest.mark.parametrize("dist_name", ["uniform", "zipf", "const", "sortedswap"])
@pytest.mark.parametrize("n", [1_000_003, 1 << 22])
def test_dist_single_rank_nvls(cuda, nccl_group, mcbuf, dist_name, n):
    """Mode N (histogram prefix written into the multicast-bound buffer, summed by
    the switch, own range expanded) on one rank equals the oracle sort."""
    keys = datagen.gen_u16(dist_name, n, seed=5)
    out, (b, e) = fsdist.sort_keys_u16(torch.from_numpy(keys).to(cuda), mode="N", peers=mcbuf)
    assert (b, e) == (0, keys.size)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.sort_u16(keys))
