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
