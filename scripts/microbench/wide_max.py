"""Wide sorts at the largest sizes one B200 holds, checked on the device by the
invariants that pin the unique stable result (sorted; values a permutation;
keys[vals] == sorted keys; equal keys keep increasing values).  Timed once
after one warm-up call.  Usage: wide_max.py [pairs_log2 [keys_log2]]."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
plog = int(sys.argv[1]) if len(sys.argv) > 1 else 31
klog = int(sys.argv[2]) if len(sys.argv) > 2 else 32
SIGN = torch.iinfo(torch.int64).min


def timed(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); r = fn(); b.record(); torch.cuda.synchronize()
    return r, a.elapsed_time(b)


def sorted_u64(x):
    y = x.view(torch.int64) ^ SIGN
    return bool((y[1:] >= y[:-1]).all().item())


for key_bits in ((64, 40) if plog else ()):
    n = 1 << plog
    k = torch.empty(n, dtype=torch.uint64, device=dev)
    v = torch.empty(n, dtype=torch.uint32, device=dev)
    datagen.gen_u64_device(k.data_ptr(), n, seed=3, stream=s, key_bits=key_bits)
    datagen.iota_u32_device(v.data_ptr(), n, stream=s)
    (ko, vo), ms = timed(lambda: fs.sort_pairs(k, v, key_bits=key_bits))
    ok = sorted_u64(ko)
    idx = vo.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    mark = torch.zeros(n, dtype=torch.uint8, device=dev)
    mark[idx] = 1
    ok &= bool(mark.all().item()); del mark
    ok &= bool((k.view(torch.int64)[idx] == ko.view(torch.int64)).all().item())
    ko64 = ko.view(torch.int64)
    same = ko64[1:] == ko64[:-1]
    ok &= bool((~same | (idx[1:] > idx[:-1])).all().item())
    print(f"pairs n=2^{plog} key_bits={key_bits}: {ms:9.2f} ms  {n / ms / 1e6:7.2f} Gpairs/s  ok={ok}", flush=True)
    del k, v, ko, vo, ko64, idx, same
    torch.cuda.empty_cache()

for dt, gen in ((torch.uint32, datagen.gen_u32_device), (torch.uint64, datagen.gen_u64_device)):
    n = 1 << klog
    k = torch.empty(n, dtype=dt, device=dev)
    gen(k.data_ptr(), n, seed=5, stream=s)
    print(f"keys {str(dt)[6:]} n=2^{klog}: sorting", flush=True)
    out, ms = timed(lambda: fs.sort_keys(k))
    print(f"keys {str(dt)[6:]} n=2^{klog}: sorted in {ms:.2f} ms, checking", flush=True)
    # checked in chunks of 2^28 (torch ops on > 2^31 elements are slow)
    C = 1 << 28
    ok = True
    hk = torch.zeros(65536, dtype=torch.int64, device=dev); ho = torch.zeros_like(hk)
    sk = so = 0
    prev = None
    for c0 in range(0, n, C):
        if dt == torch.uint32:
            a = k[c0:c0 + C].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            b = out[c0:c0 + C].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            sh = 16
        else:
            a = k[c0:c0 + C].view(torch.int64) ^ SIGN
            b = out[c0:c0 + C].view(torch.int64) ^ SIGN
            sh = 48
        ok &= bool((b[1:] >= b[:-1]).all().item()) and (prev is None or bool((b[0] >= prev).item()))
        prev = b[-1]
        hk += torch.bincount(((a >> sh) & 0xFFFF), minlength=65536)
        ho += torch.bincount(((b >> sh) & 0xFFFF), minlength=65536)
        sk += int((a & 0xFFFFFFF).sum().item()); so += int((b & 0xFFFFFFF).sum().item())
    ok &= bool((hk == ho).all().item()) and sk == so
    print(f"keys {str(dt)[6:]} n=2^{klog}: {ms:9.2f} ms  {n / ms / 1e6:7.2f} Gkeys/s  ok={ok}", flush=True)
    del k, out, hk, ho
    torch.cuda.empty_cache()
