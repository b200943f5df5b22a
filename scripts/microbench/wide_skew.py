"""Time fs_sort_pairs_u64_u32 on skewed 64-bit key distributions (oversize 16-bit
bins: the MSD recursion; repeated keys: the per-bin sort's slow path) for each
library in scripts/microbench/variants/*.so (or the in-tree library), checking
the result's order, that it is a permutation of the input pairs and stability.
n = argv[1] (default 2^28); argv[2] = comma-separated kinds: uniform, hot16x25,
hot1x50, clustered, lt2^B (keys < 2^B), dupM (each key ~M times, M a power of 2)."""
import ctypes, glob, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream


def make(kind):
    k = torch.empty(n, dtype=torch.uint64, device=dev)
    datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
    ki = k.view(torch.int64)
    r = torch.empty(n, dtype=torch.uint64, device=dev)
    datagen.gen_u64_device(r.data_ptr(), n, seed=1, stream=s)
    ri = r.view(torch.int64)
    low48 = ki & ((1 << 48) - 1)
    if kind == "uniform":
        return k
    if kind == "hot16x25":   # 25% of the keys in 16 hot 16-bit bins
        hot = (ri & 3) == 0
        top = ((ri >> 8) & 15) * 0x0F0F + 0x1234
        ki[:] = torch.where(hot, (top << 48) | low48, ki)
    elif kind == "hot1x50":  # half the keys in one bin
        hot = (ri & 1) == 0
        ki[:] = torch.where(hot, (0x7777 << 48) | low48, ki)
    elif kind.startswith("lt2^"):  # a common zero prefix: keys < 2^b
        b = int(kind[4:])
        ki[:] = ki & ((1 << b) - 1)
    elif kind.startswith("dup"):  # every key repeated ~m times: m = 8 -> "dup8" (2^29 / 8 distinct values)
        m = int(kind[3:])
        ki[:] = ki[ri & (n // m - 1)]
    elif kind == "clustered":  # 64 clusters, each 2^-8 wide in the key space (about 256 bins each)
        c = (ri & 63) * 0x0400_0000_0000_0000 // 1
        ki[:] = (c + (ki & ((1 << 56) - 1)))
    return k


kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["uniform", "hot16x25", "hot1x50", "clustered", "lt2^56", "lt2^48", "lt2^40"]
libs = sorted(glob.glob(os.path.join(ROOT, "scripts/microbench/variants/*.so"))) or \
    [os.path.join(ROOT, "paper_2605_10390_b200/libfractalsort.so")]
for path in libs:
    L = ctypes.CDLL(path)
    L.fs_sort_pairs_u64_u32_temp_bytes.restype = ctypes.c_size_t
    L.fs_sort_pairs_u64_u32_temp_bytes.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.fs_sort_pairs_u64_u32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                                                ctypes.c_size_t, ctypes.c_void_p]
    L.fs_set_phase_events.argtypes = [ctypes.c_void_p, ctypes.c_int]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(16)]
    for e in evs:
        e.record()
    harr = (ctypes.c_void_p * 16)(*[e.cuda_event for e in evs])
    temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)
    for kind in kinds:
        k = make(kind)
        v = torch.empty(n, dtype=torch.uint32, device=dev)
        datagen.iota_u32_device(v.data_ptr(), n, stream=s)
        ko, vo = torch.empty_like(k), torch.empty_like(v)
        ts = []
        for r in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if r == 4:
                L.fs_set_phase_events(harr, 16)
            rc = L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64,
                                         temp.data_ptr(), temp.numel(), s)
            b.record()
            L.fs_set_phase_events(None, 0)
            torch.cuda.synchronize()
            assert rc == 0, rc
            if r >= 2:
                ts.append(a.elapsed_time(b))
        kk = ko.view(torch.int64) ^ torch.iinfo(torch.int64).min
        ordered = bool((kk[1:] >= kk[:-1]).all().item())
        # stability + permutation: the values are the arrival indices
        vi = vo.long()
        perm = bool((torch.bincount(vi, minlength=n) == 1).all().item()) and bool((ko.view(torch.int64) == k.view(torch.int64)[vi]).all().item())
        eq = kk[1:] == kk[:-1]
        stable = bool((vi[1:][eq] > vi[:-1][eq]).all().item())
        print(f"{os.path.basename(path):24s} {kind:10s} {statistics.median(ts):8.3f} ms  "
              f"{n / statistics.median(ts) / 1e6:7.2f} Gpairs/s  ordered={ordered} perm={perm} stable={stable}  "
              + " ".join(f"{nm}={evs[i].elapsed_time(evs[i + 1]):.2f}" for i, nm in
                         enumerate(["hist", "L1", "L2", "k_heavy", "local"])) + f" lsd={evs[5].elapsed_time(evs[15]):.2f}",
              flush=True)
        del k, v, ko, vo
    del temp
    torch.cuda.empty_cache()
