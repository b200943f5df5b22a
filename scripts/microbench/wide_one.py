"""Sort n (u64, u32) pairs `reps` times through the binding (for ncu launch lists)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 15
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
k = torch.empty(n, dtype=torch.uint64, device=dev); v = torch.empty(n, dtype=torch.uint32, device=dev)
datagen.gen_u64_device(k.data_ptr(), n, seed=1, stream=s); datagen.iota_u32_device(v.data_ptr(), n, stream=s)
for _ in range(reps):
    ko, vo = fs.sort_pairs(k, v)
torch.cuda.synchronize()
print("done", n)
