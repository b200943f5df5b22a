"""Small end-to-end run of every C-ABI entry point (for compute-sanitizer and quick checks).

Usage: python scripts/sanity_small.py   (exits non-zero on any mismatch)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_10390_b200 as fs  # noqa: E402


def main() -> int:
    dev = torch.device("cuda", 0)
    bad = 0
    for n in [1, 33, 70_001, 300_007]:
        for dist in ["uniform", "zipf", "const", "sortedswap"]:
            k = datagen.gen_u16(dist, n, seed=n)
            out = fs.sort_keys(torch.from_numpy(k).to(dev)).cpu().numpy()
            if not np.array_equal(out, oracle.sort_u16(k)):
                print("u16 mismatch", n, dist)
                bad += 1
    k = datagen.gen_u16("uniform", 200_003, seed=3)
    h = fs.histogram_u16(torch.from_numpy(k).to(dev)).cpu().numpy().astype(np.uint64)
    bad += not np.array_equal(h, oracle.histogram_u16(k))
    P = fs.exclusive_scan(torch.from_numpy(h.astype(np.int64)).to(dev)).cpu().numpy().astype(np.uint64)
    bad += not np.array_equal(P, oracle.exclusive_scan(h))
    e = fs.expand_u16(torch.from_numpy(P.astype(np.int64)).to(dev), 1000, 90_000).cpu().numpy()
    bad += not np.array_equal(e, oracle.reconstruct_counts_u16(h, 1000, 90_000))
    for n in [1, 5000, 70_001]:
        k64 = datagen.gen_u64(n, seed=n)
        v = datagen.iota_u32(n)
        ko, vo = fs.sort_pairs(torch.from_numpy(k64).to(dev), torch.from_numpy(v).to(dev))
        ek, ev = oracle.sort_pairs_u64_u32(k64, v)
        if not (np.array_equal(ko.cpu().numpy(), ek) and np.array_equal(vo.cpu().numpy(), ev)):
            print("pairs mismatch", n)
            bad += 1
        k32 = datagen.gen_u32(n, seed=n)
        if not np.array_equal(fs.sort_keys(torch.from_numpy(k32).to(dev)).cpu().numpy(), oracle.sort_keys_u32(k32)):
            print("u32 mismatch", n)
            bad += 1
    H = np.stack([oracle.histogram_u16(datagen.gen_u16("zipf", 5000 + r, seed=r)) for r in range(3)])
    s = fs.send_counts(torch.from_numpy(H.astype(np.int64)).to(dev), 1).cpu().numpy().astype(np.uint64)
    bad += not np.array_equal(s, oracle.send_counts(H, 1))
    # MSD path with local sorts (bins of ~4K keys: k_local_sort), an oversize bin
    # (30,000 keys under one 16-bit prefix: k_heavy recursion), and uneven
    # first-level buckets
    for n, hot in ((400_003, 0), (200_003, 30_000)):
        k64 = datagen.gen_u64(n, seed=7)
        if hot:
            k64[:hot] = (k64[:hot] & np.uint64((1 << 48) - 1)) | np.uint64(0x4D2 << 48)
        else:
            k64 = (k64 & np.uint64((1 << 48) - 1)) | ((k64 >> np.uint64(48)) % np.uint64(100) << np.uint64(48))
        v = datagen.iota_u32(n)
        ko, vo = fs.sort_pairs(torch.from_numpy(k64).to(dev), torch.from_numpy(v).to(dev))
        ek, ev = oracle.sort_pairs_u64_u32(k64, v)
        if not (np.array_equal(ko.cpu().numpy(), ek) and np.array_equal(vo.cpu().numpy(), ev)):
            print("pairs (local / heavy) mismatch", n, hot)
            bad += 1
    # the fused peer expansion, 3 virtual ranks on one GPU (fs_expand_to_peers_u16)
    kp = datagen.gen_u16("zipf", 200_003, seed=5)
    cuts = [0, 50_000, 120_000, 200_003]
    hist_all = torch.stack([fs.histogram_u16(torch.from_numpy(kp[cuts[r]:cuts[r + 1]].copy()).to(dev))
                            for r in range(3)])
    bounds = [(200_003 * d) // 3 for d in range(4)]
    bufs = [torch.empty(bounds[d + 1] - bounds[d], dtype=torch.uint16, device=dev) for d in range(3)]
    for g in range(3):
        fs.expand_to_peers_u16(hist_all, g, bufs)
    bad += not np.array_equal(np.concatenate([b.cpu().numpy() for b in bufs]), oracle.sort_u16(kp))
    # order-statistic service: levels, packed export, GetItem / GetIndex
    kt = datagen.gen_u16("gauss", 50_001, seed=2)
    levels = fs.trie_levels(fs.histogram_u16(torch.from_numpy(kt).to(dev)), 16)
    t = fs.trie_pack(levels, 16, 50_001, 2)
    sk = np.sort(kt)
    r = torch.arange(0, 50_001, 997, dtype=torch.int64, device=dev)
    bad += not np.array_equal(fs.get_item(t, r).cpu().numpy(), sk[r.cpu().numpy()].astype(np.int64))
    vq = torch.arange(0, 65536, 613, dtype=torch.int64, device=dev)
    bad += not np.array_equal(fs.get_index(t, vq).cpu().numpy(), np.searchsorted(sk, vq.cpu().numpy(), side="left"))
    kh = datagen.gen_u16("gauss", 100_001, seed=1)
    oh = fs.sort_keys_u16_host(torch.from_numpy(kh), batch=30_000).numpy()
    bad += not np.array_equal(oh, oracle.sort_u16(kh))
    torch.cuda.synchronize()
    print("sanity_small:", "OK" if bad == 0 else f"{bad} FAILURES")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
