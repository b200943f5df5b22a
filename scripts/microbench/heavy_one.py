"""One fs_sort_pairs_u64_u32 call on a skewed distribution (for ncu captures of
the MSD recursion).  argv: kind (hot1x50 | hot16x25 | clustered), n."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
kind = sys.argv[1] if len(sys.argv) > 1 else "hot1x50"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
k = torch.empty(n, dtype=torch.uint64, device=dev)
datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
r = torch.empty(n, dtype=torch.uint64, device=dev)
datagen.gen_u64_device(r.data_ptr(), n, seed=1, stream=s)
ki, ri = k.view(torch.int64), r.view(torch.int64)
low48 = ki & ((1 << 48) - 1)
if kind == "hot1x50":
    ki[:] = torch.where((ri & 1) == 0, (0x7777 << 48) | low48, ki)
elif kind == "hot16x25":
    ki[:] = torch.where((ri & 3) == 0, ((((ri >> 8) & 15) * 0x0F0F + 0x1234) << 48) | low48, ki)
elif kind.startswith("dup"):  # every key repeated ~M times ("dup64")
    ki[:] = ki[ri & (n // int(kind[3:]) - 1)]
elif kind == "clustered":
    ki[:] = (ri & 63) * 0x0400_0000_0000_0000 + (ki & ((1 << 56) - 1))
v = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32)
for _ in range(2):
    ko, vo = fs.sort_pairs(k, v)
torch.cuda.synchronize()
print("ok")
