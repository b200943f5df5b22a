"""fs_sort_pairs_u64_u32 at sizes from 2^15 to 2^29 pairs for each library variant in
scripts/microbench/variants/*.so (median of 20, CUDA events; sortedness checked)."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
SIZES = [int(x) for x in sys.argv[1:]] or [1 << 15, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 29]
inputs = {}
for n in SIZES:
    k = torch.empty(n, dtype=torch.uint64, device=dev); v = torch.empty(n, dtype=torch.uint32, device=dev)
    datagen.gen_u64_device(k.data_ptr(), n, seed=1, stream=s); datagen.iota_u32_device(v.data_ptr(), n, stream=s)
    inputs[n] = (k, v, torch.empty_like(k), torch.empty_like(v))
for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    line = f"{os.path.basename(path):14s}"
    for n, (k, v, ko, vo) in inputs.items():
        temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)
        f = lambda: L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64,
                                            temp.data_ptr(), temp.numel(), s)
        for _ in range(3): f()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(x.elapsed_time(y) for x, y in ts)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        t2 = a.elapsed_time(b) / 20  # back to back
        kk = ko.view(torch.int64) ^ torch.iinfo(torch.int64).min
        ok = bool((kk[1:] >= kk[:-1]).all().item())
        line += f"  2^{n.bit_length() - 1}:{t * 1e3:8.1f}/{t2 * 1e3:.1f}us{'' if ok else '(BAD)'}"
        del temp
    print(line, flush=True)
