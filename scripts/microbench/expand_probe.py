"""Where the time of the expansion at c2 goes: k_expand16 alone (two-level prefix
from fs_histogram_prefix_u16), against torch's fill_ / zero_ of the same 512 MiB
(pure HBM writes) and a 2 GiB / 8 GiB expansion (steady-state rate).  Prints
median microseconds of 50 launches each (CUDA events around every launch)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream


def t(fn, reps=50):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    x = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return x[len(x) // 2]


for n in (1 << 28, 1 << 30, 1 << 32):
    k = torch.empty(n, dtype=torch.uint16, device=dev)
    datagen.gen_u16_device(k.data_ptr(), "uniform", n, seed=0, stream=s)
    pre = fs.histogram_prefix_u16(k)
    out = torch.empty_like(k)
    te = t(lambda: fs.expand_prefix_u16(pre, 0, n, out))
    tf = t(lambda: out.fill_(7))
    tz = t(lambda: out.zero_())
    gb = 2 * n / 1e9
    print(f"n=2^{n.bit_length()-1}: expand16 {te:8.2f} us ({gb/te*1e6:6.0f} GB/s)  fill_ {tf:8.2f} ({gb/tf*1e6:6.0f})  "
          f"zero_ {tz:8.2f} ({gb/tz*1e6:6.0f})", flush=True)
    del k, out, pre
    torch.cuda.empty_cache()
