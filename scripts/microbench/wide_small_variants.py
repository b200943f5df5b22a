"""Latency of fs_sort_pairs_u64_u32 at small n for each library in scripts/microbench/variants/*.so."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1000, 65536, 1 << 18, 1 << 20, 1 << 21]
for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    for n in sizes:
        k = torch.empty(n, dtype=torch.uint64, device=dev)
        datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
        v = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32)
        ko, vo = torch.empty_like(k), torch.empty_like(v)
        temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)
        f = lambda: L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64, temp.data_ptr(), temp.numel(), s)
        for _ in range(3): f()
        ts = []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        kk = ko.view(torch.int64) ^ torch.iinfo(torch.int64).min
        ok = bool((kk[1:] >= kk[:-1]).all().item()) and bool((ko.view(torch.int64) == k.view(torch.int64)[vo.long()]).all().item())
        print(f"{os.path.basename(path):20s} n={n:9d} {statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3:9.1f} us ok={ok}", flush=True)
        del k, v, ko, vo, temp
