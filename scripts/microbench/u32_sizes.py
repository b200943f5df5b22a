"""fs_sort_keys_u32 at a few sizes (median of 20, CUDA events, through the Python binding)."""
import os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
for n in [1 << 20, 1 << 24, 1 << 28]:
    k = torch.empty(n, dtype=torch.uint32, device=dev)
    datagen.gen_u32_device(k.data_ptr(), n, seed=0, stream=s)
    out = torch.empty_like(k)
    for _ in range(3): fs.sort_keys(k, out=out)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fs.sort_keys(k, out=out); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    t = statistics.median(x.elapsed_time(y) for x, y in ts)
    ok = bool((out[1:].view(torch.int32).to(torch.int64) & 0xFFFFFFFF >= (out[:-1].view(torch.int32).to(torch.int64) & 0xFFFFFFFF)).all().item())
    print(f"u32 n={n:10d} {t * 1e3:9.1f} us  {n / t / 1e6:7.1f} Gkeys/s  {n * 28 / t / 1e9 * 1e3 / 1e3:6.2f} TB/s@28B/key sorted={ok}", flush=True)
