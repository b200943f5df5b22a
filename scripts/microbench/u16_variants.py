"""Time fs_sort_keys_u16 on c2 (2^28 uniform u16) for each library variant in
scripts/microbench/variants/*.so: median of 30 timed sorts (CUDA events)."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

dist = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
k = torch.empty(n, dtype=torch.uint16, device=dev)
if dist == "sortedswap":
    k.copy_(torch.from_numpy(datagen.gen_u16("sortedswap", n, seed=0)))
else:
    datagen.gen_u16_device(k.data_ptr(), dist, n, seed=0, stream=s)
out = torch.empty_like(k)
for rnd in range(1):
  for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_keys_u16_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_keys_u16_temp_bytes.argtypes = [ctypes.c_uint64]
    L.fs_sort_keys_u16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
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
    ok = bool((out[1:].to(torch.int32) >= out[:-1].to(torch.int32)).all().item())
    # back to back: one event pair around 100 calls (as bench.py times its steps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        L.fs_sort_keys_u16(k.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s)
    b.record(); torch.cuda.synchronize()
    b2b = a.elapsed_time(b) * 1e3 / 100
    print(f"{dist:10s} {os.path.basename(path):24s} median {t[len(t)//2]:7.2f} us  min {t[0]:7.2f}  b2b {b2b:7.2f}  sorted={ok}", flush=True)
