"""Back-to-back u16 sorts at small n: plain stream launches vs one CUDA graph
(captured fs_sort_keys_u16 calls) replayed; checks the graph's output."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
from paper_2605_10390_b200 import _lib

dev = torch.device("cuda", 0)
L = fs.lib()
for n in [int(x) for x in (sys.argv[1:] or [str(1 << 16), str(1 << 18), str(1 << 20), str(1 << 22)])]:
    k = torch.empty(n, dtype=torch.uint16, device=dev)
    s = torch.cuda.Stream(dev)
    datagen.gen_u16_device(k.data_ptr(), "uniform", n, seed=0, stream=s.cuda_stream)
    out = torch.empty_like(k)
    temp = torch.empty(L.fs_sort_keys_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
    reps = 200

    def call(st):
        _lib.check(L.fs_sort_keys_u16(k.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), st),
                   "fs_sort_keys_u16")
    with torch.cuda.stream(s):
        for _ in range(5):
            call(s.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            call(s.cuda_stream)
        b.record(s)
    torch.cuda.synchronize()
    t_plain = a.elapsed_time(b) * 1e3 / reps
    g = torch.cuda.CUDAGraph()
    per = 20
    with torch.cuda.graph(g, stream=s):
        for _ in range(per):
            call(s.cuda_stream)
    out.zero_()
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        ok = bool(torch.equal(out.view(torch.int16).to(torch.int32) & 0xFFFF,
                              torch.sort(k.view(torch.int16).to(torch.int32) & 0xFFFF).values))
        a.record(s)
        for _ in range(reps // per):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    t_graph = a.elapsed_time(b) * 1e3 / reps
    print(f"n={n:9d}  stream {t_plain:7.2f} us/sort   graph {t_graph:7.2f} us/sort   exact={ok}", flush=True)
