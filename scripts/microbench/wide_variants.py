"""Time the c5 sort (2^29 u64/u32 pairs, MSD path) for each library variant in
scripts/microbench/variants/*.so; prints per-phase milliseconds (CUDA events)."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 29
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
k = torch.empty(n, dtype=torch.uint64, device=dev); v = torch.empty(n, dtype=torch.uint32, device=dev)
datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s); datagen.iota_u32_device(v.data_ptr(), n, stream=s)
ko, vo = torch.empty_like(k), torch.empty_like(v)
names = ["hist", "L1", "L2", "heavy", "local", "lsd"]
for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.fs_set_phase_events.argtypes = [ctypes.c_void_p, ctypes.c_int]
    temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(16)] for _ in range(4)]
    for row in ev:
        for e in row: e.record()
    arrs = [(ctypes.c_void_p * 16)(*[e.cuda_event for e in row]) for row in ev]
    torch.cuda.synchronize()
    for r in range(6):
        h = arrs[r - 2] if r >= 2 else None
        if h is not None: L.fs_set_phase_events(h, 16)
        rc = L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64, temp.data_ptr(), temp.numel(), s)
        L.fs_set_phase_events(None, 0)
        assert rc == 0, rc
    torch.cuda.synchronize()
    ph = [statistics.median(row[i].elapsed_time(row[i + 1]) for row in ev) for i in range(5)]
    lsd = statistics.median(row[5].elapsed_time(row[15]) for row in ev)
    tot = statistics.median(row[0].elapsed_time(row[15]) for row in ev)
    kk = ko.view(torch.int64) ^ torch.iinfo(torch.int64).min
    ok = bool((kk[1:] >= kk[:-1]).all().item())
    print(f"{os.path.basename(path):28s} total {tot:7.3f}  " + "  ".join(f"{nm} {x:6.3f}" for nm, x in zip(names, ph + [lsd])) + f"  sorted={ok}", flush=True)
    del temp; torch.cuda.empty_cache()
