"""Host-buffer sorts (fs_sort_keys_u16_host) back to back on two streams, as
bench.py's e2e leg, for several batch sizes: Gkeys/s per batch size."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
from paper_2605_10390_b200 import _lib

n = 1 << 28
dev = torch.device("cuda", 0)
L = fs.lib()
k = torch.empty(n, dtype=torch.uint16, device=dev)
datagen.gen_u16_device(k.data_ptr(), "uniform", n, seed=0, stream=torch.cuda.current_stream().cuda_stream)
host_in = k.cpu().pin_memory()
outs = [torch.empty(n, dtype=torch.uint16).pin_memory() for _ in range(3)]
for nstreams in (2, 3):
    for lb in (22, 23, 24, 25, 26):
        B = 1 << lb
        streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        works = [torch.empty(L.fs_sort_keys_u16_host_work_bytes(n, B), dtype=torch.uint8, device=dev)
                 for _ in range(nstreams)]

        def block(steps):
            cur = torch.cuda.current_stream(dev)
            for st in streams:
                st.wait_stream(cur)
            for i in range(steps):
                j = i % nstreams
                _lib.check(L.fs_sort_keys_u16_host(host_in.data_ptr(), outs[j].data_ptr(), n, B, works[j].data_ptr(),
                                                   works[j].numel(), streams[j].cuda_stream), "host sort")
            for st in streams:
                cur.wait_stream(st)
        block(2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        block(10)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"streams {nstreams} batch 2^{lb}: {ms:7.2f} ms/sort  {n / ms / 1e6:6.2f} Gkeys/s", flush=True)
        del works
