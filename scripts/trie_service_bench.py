"""Order-statistic service on c2's histogram: times the
histogram of 2^28 uint16 keys, the dense trie levels, the tapered bit-packed
export and 2^20 batched GetItem / GetIndex queries on the packed trie (CUDA
events, median of 20), and checks 1,000 sampled answers against the oracle."""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_10390_b200 as fs  # noqa: E402


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    n, q = 1 << 28, 1 << 20
    dev = torch.device("cuda", 0)
    k = torch.empty(n, dtype=torch.uint16, device=dev)
    datagen.gen_u16_device(k.data_ptr(), "zipf", n, seed=0, stream=torch.cuda.current_stream().cuda_stream)
    hist = fs.histogram_u16(k)
    levels = fs.trie_levels(hist, 16)
    t = fs.trie_pack(levels, 16, n, 1)
    rng = np.random.default_rng(0)
    ranks = torch.from_numpy(rng.integers(0, n, q).astype(np.int64)).to(dev)
    values = torch.from_numpy(rng.integers(0, 65536, q).astype(np.int64)).to(dev)
    out = {
        "workload": "c3a keys (2^28 uint16, Zipf s=1.2), queries: 2^20 random ranks / values",
        "histogram_ms": round(timed(lambda: fs.histogram_u16(k, hist=hist)), 4),
        "trie_levels_ms": round(timed(lambda: fs.trie_levels(hist, 16)), 4),
        "trie_pack_ms": round(timed(lambda: fs.trie_pack(levels, 16, n, 1)), 4),
        "get_item_ms": round(timed(lambda: fs.get_item(t, ranks)), 4),
        "get_index_ms": round(timed(lambda: fs.get_index(t, values)), 4),
        "packed_bits": int(t.bit_offsets[-1].item()),
        "dense_bits": 64 * ((1 << 17) - 1),
        "widths": [int(x) for x in t.widths.cpu().tolist()],
    }
    out["queries_per_s_get_item"] = round(q / (out["get_item_ms"] * 1e-3), 1)
    items = fs.get_item(t, ranks[:1000]).cpu().numpy()
    idx = fs.get_index(t, values[:1000]).cpu().numpy()
    lv = oracle.trie_levels(k.cpu().numpy().astype(np.uint64), 16)
    out["verified"] = bool(all(items[i] == oracle.get_item(lv, 16, int(r)) for i, r in enumerate(ranks[:1000].cpu().tolist()))
                           and all(idx[i] == oracle.get_index(lv, 16, int(v)) for i, v in enumerate(values[:1000].cpu().tolist())))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
