"""Time fs_sort_keys_u16 at c2 size for each library variant in
scripts/microbench/variants/*.so: median / min of 100 sorts (CUDA events around
each) and back-to-back (one event pair around 100 sorts), for one or more
distributions.  Every variant's output is compared with torch's sort of the same
keys (exact).  Usage: u16_variants.py [dist[,dist...]] [n]"""
import ctypes, glob, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

dists = (sys.argv[1] if len(sys.argv) > 1 else "uniform").split(",")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
paths = sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so")))
libs = []
for path in paths:
    L = ctypes.CDLL(path)
    L.fs_sort_keys_u16_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_keys_u16_temp_bytes.argtypes = [ctypes.c_uint64]
    L.fs_sort_keys_u16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_size_t, ctypes.c_void_p]
    libs.append((os.path.basename(path), L))
for dist in dists:
    k = torch.empty(n, dtype=torch.uint16, device=dev)
    if dist == "sortedswap":
        k.copy_(torch.from_numpy(datagen.gen_u16("sortedswap", n, seed=0)))
    else:
        datagen.gen_u16_device(k.data_ptr(), dist, n, seed=0, stream=s)
    want = k.to(torch.int32).sort().values
    out = torch.empty_like(k)
    for name, L in libs:
        temp = torch.empty(L.fs_sort_keys_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
        for _ in range(5):
            L.fs_sort_keys_u16(k.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s)
        ts = []
        for _ in range(100):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); L.fs_sort_keys_u16(k.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s); b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
        ok = bool(torch.equal(out.to(torch.int32), want))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(100):
            L.fs_sort_keys_u16(k.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s)
        b.record(); torch.cuda.synchronize()
        b2b = a.elapsed_time(b) * 1e3 / 100
        print(f"{dist:10s} {name:24s} median {t[len(t)//2]:7.2f} us  min {t[0]:7.2f}  b2b {b2b:7.2f}  exact={ok}",
              flush=True)
        del temp
    del k, want, out
