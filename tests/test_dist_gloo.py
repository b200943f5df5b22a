"""Multi-rank orchestration of paper_2605_10390_b200.dist on CPU: gloo process
groups (world size 2, 3, 4), one process per rank, 127.0.0.1 rendezvous.

The local steps are injected (OracleOps below, built from the oracle in tests/
only); the collectives, split sizes, output ranges and the byte-level all-to-all
are exactly dist.py's.  The concatenation of every rank's output slice must equal
the single-process oracle sort of the union of the shards.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleOps:
    """CPU stand-ins for the library calls, computed by the oracle (tests only)."""

    def histogram_u16(self, keys):
        import oracle
        return torch.from_numpy(oracle.histogram_u16(keys.numpy()).astype(np.int64))

    def histogram_prefix_u16(self, keys):
        """Two-level form: slice-local exclusive prefixes (512-bin slices) + slice totals."""
        import oracle
        P = oracle.exclusive_scan(oracle.histogram_u16(keys.numpy())).astype(np.int64)
        L = P[:65536] - np.repeat(P[0:65536:512], 512)
        tot = P[512:65537:512] - P[0:65536:512]
        return torch.from_numpy(np.concatenate([L, tot]).astype(np.int64))

    def expand_prefix_u16(self, prefix2, begin, end):
        import oracle
        p2 = prefix2.numpy().astype(np.int64)
        base = np.concatenate([[0], np.cumsum(p2[65536:])])[:128]
        P = np.concatenate([p2[:65536] + np.repeat(base, 512), [p2[65536:].sum()]]).astype(np.uint64)
        return torch.from_numpy(oracle.reconstruct_counts_u16(np.diff(P), begin, end))

    def exclusive_scan(self, hist):
        import oracle
        return torch.from_numpy(oracle.exclusive_scan(hist.numpy().astype(np.uint64)).astype(np.int64))

    def expand_u16(self, prefix, begin, end):
        import oracle
        P = prefix.numpy().astype(np.uint64)
        C = np.diff(P)
        return torch.from_numpy(oracle.reconstruct_counts_u16(C, begin, end))

    def sort_keys(self, keys):
        import oracle
        return torch.from_numpy(oracle.sort_u16(keys.numpy()))

    def send_counts(self, hist_all, g):
        import oracle
        return torch.from_numpy(oracle.send_counts(hist_all.numpy().astype(np.uint64), g).astype(np.int64))

    def expand_to_peers(self, hist_all, g, dest):
        """Rank g's keys to their global positions (P[v] + S_<g[v] + local offset) in
        the owning rank's buffer -- the definition, with the oracle's scans."""
        import oracle
        C = hist_all.numpy().astype(np.uint64)
        G = C.shape[0]
        P = oracle.exclusive_scan(C.sum(axis=0))
        S = C[:g].sum(axis=0) if g else np.zeros(C.shape[1], dtype=np.uint64)
        Pg = oracle.exclusive_scan(C[g])
        vals = oracle.reconstruct_counts_u16(C[g], 0, int(Pg[-1]))  # rank g's keys in sorted order
        v = vals.astype(np.int64)
        j = np.arange(vals.size, dtype=np.uint64)
        pos = P[v] + S[v] + j - Pg[v]
        N = int(P[-1])
        begins = np.array([(N * d) // G for d in range(G + 1)], dtype=np.uint64)
        owner = np.searchsorted(begins, pos, side="right") - 1
        for d in range(G):
            sel = owner == d
            dest[d].numpy()[(pos[sel] - begins[d]).astype(np.int64)] = vals[sel]

    def synchronize(self, device):
        pass

    # -- mode "N": the multicast buffer's halves live in FakeMulticast.store (keyed by
    #    the local address); the switch's multimem.ld_reduce sum is an all_reduce
    def histogram_prefix_u16_to(self, keys, out_ptr):
        FakeMulticast.store[out_ptr] = self.histogram_prefix_u16(keys)

    def allreduce_multicast(self, src_mc, dst, flag_mc, flag_local, target):
        assert flag_mc == flag_local + FakeMulticast.MC, "flag: multicast and local views of one word"
        assert target == dist.get_world_size() * FakeMulticast.calls, "target = G x calls on this flag"
        t = FakeMulticast.store.pop(src_mc - FakeMulticast.MC).clone()
        dist.all_reduce(t)
        dst.copy_(t)
        return dst, torch.zeros(1, dtype=torch.int32)

    def sort_pairs(self, keys, vals):
        import oracle
        k, v = oracle.sort_pairs_u64_u32(keys.numpy(), vals.numpy())
        return torch.from_numpy(k), torch.from_numpy(v)

    def bound_u64(self, sorted_keys, queries, upper):
        # a library routine stands in for fs_bound_u64 on CPU
        return torch.from_numpy(np.searchsorted(sorted_keys.numpy(), queries.numpy(),
                                                side="right" if upper else "left").astype(np.int64))

    # -- the distributed pair sort's splitter levels and fused exchange, by definition
    def histogram16_u64(self, keys, shift, width):
        d = (keys.numpy() >> np.uint64(shift)) & np.uint64((1 << width) - 1)
        return torch.from_numpy(np.bincount(d.astype(np.int64), minlength=1 << width).astype(np.int64))

    def select_bins_u64(self, keys, shift, width, bins, cap):
        k = keys.numpy()
        d = (k >> np.uint64(shift)) & np.uint64((1 << width) - 1)
        sel = k[np.isin(d, np.array(bins, dtype=np.uint64))]
        assert sel.size <= cap
        return torch.from_numpy(sel.copy())

    def sort_keys_u64(self, keys):
        import oracle
        return torch.from_numpy(oracle.sort_keys_u64(keys.numpy()))

    def digit_counts_sorted_u64(self, sorted_keys, prefixes, shift, width):
        hi = sorted_keys.numpy() >> np.uint64(shift)
        out = np.zeros((len(prefixes), 1 << width), dtype=np.int64)
        for j, p in enumerate(prefixes):
            t = (np.uint64(p) >> np.uint64(shift)) | np.arange(1 << width, dtype=np.uint64)
            out[j] = np.searchsorted(hi, t, side="right") - np.searchsorted(hi, t, side="left")
        return torch.from_numpy(out)

    def pair_exchange(self, keys, vals, splitters, G):
        return _OracleExchange(keys, vals, splitters, G)


class _OracleExchange:
    """fs_pair_classes_u64 / fs_pair_scatter_u64_u32 by their definition: class 2d for
    K_{d-1} < key < K_d, 2d + 1 for key == K_d (lowest d); class order stable; pair with
    class-order index Q in [cuts[d], cuts[d+1]) goes to dest[d][bases[d] + Q - cuts[d]]."""

    def __init__(self, keys, vals, splitters, G):
        k = keys.numpy()
        K = np.array(splitters, dtype=np.uint64)
        d = np.searchsorted(K, k, side="left")
        tie = np.zeros(k.size, dtype=bool)
        inside = d < K.size
        tie[inside] = K[d[inside]] == k[inside]
        self.cls = 2 * d + tie
        self.k, self.v, self.G = k, vals.numpy(), G

    def classes(self):
        return np.bincount(self.cls, minlength=2 * self.G - 1).astype(np.int64).tolist()

    def scatter(self, cuts, bases, dest_keys, dest_vals):
        order = np.argsort(self.cls, kind="stable")
        Q = np.arange(order.size)
        owner = np.searchsorted(np.array(cuts), Q, side="right") - 1
        for dd in range(self.G):
            sel = owner == dd
            slots = np.array(bases[dd]) + Q[sel] - cuts[dd]
            dest_keys[dd].numpy()[slots] = self.k[order[sel]]
            dest_vals[dd].numpy()[slots] = self.v[order[sel]]


class FakeMulticast:
    """CPU stand-in of dist.MulticastBuffer: the same step() contract (two halves by
    call parity, the flag's multicast/local addresses, target = G x calls) over
    made-up addresses."""
    MC = 1 << 40
    store = {}
    calls = 0

    def __init__(self, world):
        self.world = world

    def step(self):
        FakeMulticast.calls += 1
        h = FakeMulticast.calls & 1
        uc = 4096 + h * 65536 * 8
        return uc, uc + self.MC, 3 * 65536 * 8 + self.MC, 3 * 65536 * 8, self.world * FakeMulticast.calls


class SharedPeers:
    """CPU stand-in of dist.PeerBuffers: shared-memory buffers made by the parent."""

    def __init__(self, bufs):
        self.bufs = bufs

    def buffers(self, per_rank):
        assert all(b.numel() >= per_rank for b in self.bufs)
        return self.bufs


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_bounds(n_total, world, rank, uneven):
    if not uneven:
        return (n_total * rank) // world, (n_total * (rank + 1)) // world
    # deliberately uneven shards, including an empty one when world > 2
    cuts = [0] + sorted({(n_total * (3 * r + 1)) // (3 * world) for r in range(1, world)}) + [n_total]
    while len(cuts) < world + 1:
        cuts.insert(1, 0)
    return cuts[rank], cuts[rank + 1]


CASES = [(mode, d, uneven) for mode in ("B", "A", "P", "N")
         for d, uneven in (("uniform", False), ("zipf", True), ("const", False), ("sortedswap", True))]
N_TOTAL = 50_003


def worker(rank, world, port, outdir, peer_bufs):
    sys.path.insert(0, ROOT)
    import datagen
    from paper_2605_10390_b200 import dist as fsdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mc = FakeMulticast(world)   # one buffer across the mode-N cases: the halves alternate
    try:
        for ci, (mode, dist_name, uneven) in enumerate(CASES):
            b, e = shard_bounds(N_TOTAL, world, rank, uneven)
            full = datagen.gen_u16(dist_name, N_TOTAL, seed=3)
            shard = torch.from_numpy(full[b:e].copy())
            peers = SharedPeers(peer_bufs[ci]) if mode == "P" else (mc if mode == "N" else None)
            out, (ob, oe) = fsdist.sort_keys_u16(shard, mode=mode, ops=OracleOps(), peers=peers)
            np.save(os.path.join(outdir, f"out_{ci}_{rank}.npy"), out.numpy())
            np.save(os.path.join(outdir, f"range_{ci}_{rank}.npy"), np.array([ob, oe], dtype=np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_distributed_sort_matches_oracle(tmp_path, world):
    """Modes A, B, P (expand-to-peer) and N (NVLS orchestration, stand-in switch), four
    distributions (uneven and empty shards included)."""
    import datagen
    import oracle
    cap = -(-N_TOTAL // world)
    peer_bufs = [[torch.zeros(cap, dtype=torch.uint16).share_memory_() for _ in range(world)] for _ in CASES]
    mp.start_processes(worker, args=(world, free_port(), str(tmp_path), peer_bufs), nprocs=world, join=True,
                       start_method="spawn")
    for ci, (mode, dist_name, uneven) in enumerate(CASES):
        outs = [np.load(tmp_path / f"out_{ci}_{r}.npy") for r in range(world)]
        ranges = [tuple(np.load(tmp_path / f"range_{ci}_{r}.npy")) for r in range(world)]
        # exact equal-count partition (ledger 23): rank d owns [floor(dN/G), floor((d+1)N/G))
        assert ranges == [((N_TOTAL * d) // world, (N_TOTAL * (d + 1)) // world) for d in range(world)], (mode, dist_name)
        for (b, e), o in zip(ranges, outs):
            assert o.size == e - b
        want = oracle.sort_u16(datagen.gen_u16(dist_name, N_TOTAL, seed=3))
        np.testing.assert_array_equal(np.concatenate(outs), want, err_msg=f"{mode} {dist_name} world={world}")


def test_output_range_helper():
    from paper_2605_10390_b200.dist import output_range
    n = 17
    ranges = [output_range(r, 4, n) for r in range(4)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(3))
    assert sorted(e - b for b, e in ranges) == [4, 4, 4, 5]


PAIR_CASES = [("uniform", False, "A"), ("ties8", True, "A"), ("const", False, "A"), ("ties3", True, "A"),
              ("uniform", True, "P"), ("ties8", False, "P"), ("const", True, "P"), ("ties3", False, "P"),
              ("hi16", True, "P"), ("hi16", False, "A")]
N_PAIRS = 20_011


def pair_input(kind):
    import datagen
    k = datagen.gen_u64(N_PAIRS, seed=9)
    if kind == "ties8":
        k = k & np.uint64(7)          # ties straddle every rank boundary
    elif kind == "ties3":
        k = (k % np.uint64(3)) << np.uint64(62)
    elif kind == "const":
        k = np.full(N_PAIRS, 0xFEDCBA9876543210, dtype=np.uint64)
    elif kind == "hi16":              # every key in one top-16 bin: the later levels decide
        k = (k & np.uint64((1 << 48) - 1)) | np.uint64(0xBEEF << 48)
    return k, datagen.iota_u32(N_PAIRS)


def pair_worker(rank, world, port, outdir, peer_bufs):
    sys.path.insert(0, ROOT)
    from paper_2605_10390_b200 import dist as fsdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (kind, uneven, mode) in enumerate(PAIR_CASES):
            b, e = shard_bounds(N_PAIRS, world, rank, uneven)
            k, v = pair_input(kind)
            peers = (SharedPeers(peer_bufs[ci][0]), SharedPeers(peer_bufs[ci][1])) if mode == "P" else None
            (ok, ov), (ob, oe) = fsdist.sort_pairs_u64_u32(torch.from_numpy(k[b:e].copy()),
                                                           torch.from_numpy(v[b:e].copy()), ops=OracleOps(),
                                                           mode=mode, peers=peers)
            np.save(os.path.join(outdir, f"pk_{ci}_{rank}.npy"), ok.numpy())
            np.save(os.path.join(outdir, f"pv_{ci}_{rank}.npy"), ov.numpy())
            np.save(os.path.join(outdir, f"pr_{ci}_{rank}.npy"), np.array([ob, oe], dtype=np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_distributed_pairs_match_oracle(tmp_path, world):
    """Pairs, modes A (local sort, all_to_all, local sort) and P (classes, stores into
    the owners' buffers, one sort): exact splitters from one all-reduced 16-bit
    histogram per level, tie split by source rank.  The concatenated slices equal
    the oracle's stable sort of the whole input (values = arrival indices:
    stability checked), for uniform keys, few distinct keys whose ties straddle
    every boundary, constant keys and keys sharing their top 16 bits."""
    import oracle
    cap = -(-N_PAIRS // world)
    peer_bufs = [([torch.zeros(cap, dtype=torch.int64).view(torch.uint64).share_memory_() for _ in range(world)],
                  [torch.zeros(cap, dtype=torch.int32).view(torch.uint32).share_memory_() for _ in range(world)])
                 for _ in PAIR_CASES]
    mp.start_processes(pair_worker, args=(world, free_port(), str(tmp_path), peer_bufs), nprocs=world, join=True,
                       start_method="spawn")
    for ci, (kind, uneven, mode) in enumerate(PAIR_CASES):
        ks = [np.load(tmp_path / f"pk_{ci}_{r}.npy") for r in range(world)]
        vs = [np.load(tmp_path / f"pv_{ci}_{r}.npy") for r in range(world)]
        ranges = [tuple(np.load(tmp_path / f"pr_{ci}_{r}.npy")) for r in range(world)]
        assert ranges == [((N_PAIRS * d) // world, (N_PAIRS * (d + 1)) // world) for d in range(world)]
        k, v = pair_input(kind)
        ek, ev = oracle.sort_pairs_u64_u32(k, v)
        np.testing.assert_array_equal(np.concatenate(ks), ek, err_msg=f"{kind} {mode} world={world}")
        np.testing.assert_array_equal(np.concatenate(vs), ev, err_msg=f"{kind} {mode} world={world}")


@pytest.mark.parametrize("G", [2, 3, 5, 8])
@pytest.mark.parametrize("kind", ["uniform", "few", "const", "hi16"])
def test_splitter_levels_and_cuts_single_process(G, kind):
    """dist.splitter_level1 / splitter_refine / pair_cuts without collectives: the
    per-rank histograms are summed here.  The splitters must be exactly the keys
    at the rank boundaries of the stable global order, and every rank's cuts must
    select exactly the elements the stable global sort gives each owner, in that
    owner's order (lower rank first for ties)."""
    import datagen
    from paper_2605_10390_b200 import dist as fsd
    n = 30_011
    k = datagen.gen_u64(n, seed=G)
    if kind == "few":
        k = k % np.uint64(5)
    elif kind == "const":
        k = np.full(n, 77, dtype=np.uint64)
    elif kind == "hi16":
        k = (k & np.uint64((1 << 48) - 1)) | np.uint64(0xABCD << 48)
    cuts_in = [0] + sorted(int(x) for x in datagen.gen_u64(G - 1, seed=1) % np.uint64(n)) + [n]
    shards = [k[cuts_in[r]:cuts_in[r + 1]] for r in range(G)]
    levels = fsd._levels(64)
    bounds = [(n * d) // G for d in range(1, G)]
    s1, w1 = levels[0]
    H = sum(np.bincount((s >> np.uint64(s1)).astype(np.int64), minlength=1 << w1) for s in shards)
    K, L = fsd.splitter_level1(H, bounds, s1)
    for shift, width in levels[1:]:
        Hl = np.zeros((G - 1, 1 << width), dtype=np.int64)
        for s in shards:
            hi = np.sort(s) >> np.uint64(shift)
            for j, p in enumerate(K):
                t = (np.uint64(p) >> np.uint64(shift)) | np.arange(1 << width, dtype=np.uint64)
                Hl[j] += np.searchsorted(hi, t, side="right") - np.searchsorted(hi, t, side="left")
        fsd.splitter_refine(Hl, bounds, K, L, shift)
    order = np.argsort(k, kind="stable")                      # the stable global order
    assert K == [int(k[order[b]]) for b in bounds]
    assert L == [int((k < np.uint64(x)).sum()) for x in K]
    # classes per rank, then every rank's cuts
    Ka = np.array(K, dtype=np.uint64)
    T_all = []
    cls_all = []
    for s in shards:
        d = np.searchsorted(Ka, s, side="left")
        tie = np.zeros(s.size, dtype=bool)
        inside = d < Ka.size
        tie[inside] = Ka[d[inside]] == s[inside]
        c = 2 * d + tie
        cls_all.append(c)
        T_all.append(np.bincount(c, minlength=2 * G - 1))
    cuts_all = fsd.pair_cuts(np.array(T_all), K, L, bounds, [s.size for s in shards])
    owner_of = np.empty(n, dtype=np.int64)                   # global index -> owner, by the stable sort
    for d in range(G):
        owner_of[order[(n * d) // G:(n * (d + 1)) // G]] = d
    for r, (s, c) in enumerate(zip(shards, cls_all)):
        perm = np.argsort(c, kind="stable") + cuts_in[r]     # class order, as global indices
        for d in range(G):
            part = perm[cuts_all[r][d]:cuts_all[r][d + 1]]
            assert np.all(owner_of[part] == d), (r, d)
            assert part.size == int((owner_of[cuts_in[r]:cuts_in[r + 1]] == d).sum())


def _fd_worker(rank, world, port, path):
    sys.path.insert(0, ROOT)
    from paper_2605_10390_b200 import dist as fsdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = os.open(path, os.O_RDONLY) if rank == 0 else None
        got = fsdist.share_fd(fd, None)
        assert os.pread(got, 64, 0) == b"multicast handle stand-in"   # the same open file (shared offset: pread)
        if rank:
            assert got != fd
        os.close(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_share_fd(tmp_path, world):
    """dist.share_fd (how MulticastBuffer hands rank 0's POSIX multicast handle to
    the other ranks): every rank ends up with a descriptor of rank 0's open file."""
    path = tmp_path / "h"
    path.write_bytes(b"multicast handle stand-in")
    mp.start_processes(_fd_worker, args=(world, free_port(), str(path)), nprocs=world, join=True,
                       start_method="spawn")


def test_multicast_step_contract():
    """MulticastBuffer.step's addresses: the two halves alternate by call parity
    (consecutive calls never share a half), the flag's multicast and local
    addresses are the same offset in the two mappings, and the target is G x
    calls modulo 2^32 (wrap-safe in the kernel)."""
    from paper_2605_10390_b200.dist import multicast_step
    uc, mc, half, flag = 0x7F0000000000, 0x7E0000000000, 525_312, 2 * 525_312
    prev = None
    for calls in range(1, 9):
        u, m, fm, fl, tgt = multicast_step(calls, 8, uc, mc, half, flag)
        assert u - uc == m - mc and (u - uc) in (0, half)
        assert fm - mc == fl - uc == flag
        assert tgt == 8 * calls
        assert u != prev
        prev = u
    assert multicast_step(1 << 30, 8, uc, mc, half, flag)[4] == (8 << 30) & 0xFFFFFFFF
