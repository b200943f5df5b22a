"""Cold vs L2-warm cost of k_local_sort: variants built with -DFS_LOCAL_PROBE=NB
re-sort the first NB bins of a c5 sort twice after the pipeline (the first time
from DRAM, the second from the lines the first just wrote); prints both times
and the per-bin cost.  Sizes the upper bound of an L2-resident level-2 ->
local-sort handoff."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

n = 1 << 29
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
k = torch.empty(n, dtype=torch.uint64, device=dev); v = torch.empty(n, dtype=torch.uint32, device=dev)
datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s); datagen.iota_u32_device(v.data_ptr(), n, stream=s)
ko, vo = torch.empty_like(k), torch.empty_like(v)
for path in sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/p*.so"))):
    L = ctypes.CDLL(path)
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)
    out = (ctypes.c_float * 2)()
    cold, warm = [], []
    for r in range(8):
        rc = L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64, temp.data_ptr(), temp.numel(), s)
        assert rc == 0, rc
        torch.cuda.synchronize()
        L.fs_probe_local_ms(out)
        if r >= 2: cold.append(out[0]); warm.append(out[1])
    nb = int(os.path.basename(path)[1:-3])
    kk = ko.view(torch.int64) ^ torch.iinfo(torch.int64).min
    ok = bool((kk[1:] >= kk[:-1]).all().item())
    c, w = statistics.median(cold), statistics.median(warm)
    print(f"bins {nb:6d} ({nb * 8192 * 12 / 1e6:6.1f} MB)  cold {c * 1e3:8.1f} us  warm {w * 1e3:8.1f} us  "
          f"per-bin-slot cold {c * 1e3 / nb * 296:6.2f} warm {w * 1e3 / nb * 296:6.2f} us  sorted={ok}", flush=True)
    del temp; torch.cuda.empty_cache()
