"""Time fs_sort_keys_u32 (2^28 and 2^24 uniform keys) and fs_sort_pairs_u64_u32
(2^28 pairs) for each library variant in scripts/microbench/variants/*.so
(median of 10, CUDA events)."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts)


inputs = {}
for n in (1 << 24, 1 << 28):
    k = torch.empty(n, dtype=torch.uint32, device=dev)
    datagen.gen_u32_device(k.data_ptr(), n, seed=0, stream=s)
    inputs[n] = (k, torch.empty_like(k))
n2 = 1 << 28
pk = torch.empty(n2, dtype=torch.uint64, device=dev); pv = torch.empty(n2, dtype=torch.uint32, device=dev)
datagen.gen_u64_device(pk.data_ptr(), n2, seed=0, stream=s); datagen.iota_u32_device(pv.data_ptr(), n2, stream=s)
pko, pvo = torch.empty_like(pk), torch.empty_like(pv)

for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_keys_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_keys_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_keys_u32.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    line = f"{os.path.basename(path):20s}"
    for n, (k, out) in inputs.items():
        temp = torch.empty(L.fs_sort_keys_u32_temp_bytes(n, 32), dtype=torch.uint8, device=dev)
        t = timed(lambda: L.fs_sort_keys_u32(k.data_ptr(), out.data_ptr(), n, 32, temp.data_ptr(), temp.numel(), s))
        kk = out.to(torch.int64) if False else out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        ok = bool((kk[1:] >= kk[:-1]).all().item())
        line += f"  u32 2^{n.bit_length() - 1} {t:7.3f} ms ok={ok}"
        del temp
    temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n2, 64), dtype=torch.uint8, device=dev)
    t = timed(lambda: L.fs_sort_pairs_u64_u32(pk.data_ptr(), pv.data_ptr(), pko.data_ptr(), pvo.data_ptr(), n2, 64,
                                             temp.data_ptr(), temp.numel(), s))
    kk = pko.view(torch.int64) ^ torch.iinfo(torch.int64).min
    ok = bool((kk[1:] >= kk[:-1]).all().item())
    line += f"  pairs 2^28 {t:7.3f} ms ok={ok}"
    del temp; torch.cuda.empty_cache()
    print(line, flush=True)
