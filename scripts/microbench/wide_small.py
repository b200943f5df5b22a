"""Latency of fs_sort_pairs_u64_u32 / fs_sort_keys_u32 at small n (median of 50, CUDA events)."""
import os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
for n in [1000, 65536, 1 << 18, 1 << 20, (1 << 22) - 1, 1 << 22]:
    k = torch.empty(n, dtype=torch.uint64, device=dev)
    datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
    v = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32)
    k32 = (k.view(torch.int64) & 0xFFFFFFFF).to(torch.int64).to(torch.uint32) if hasattr(torch, "uint32") else None
    for name, fn in [("pairs u64", lambda: fs.sort_pairs(k, v)), ("keys u64", lambda: fs.sort_keys(k))]:
        for _ in range(5): fn()
        ts = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        print(f"n={n:9d} {name:10s} {statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3:9.1f} us", flush=True)
