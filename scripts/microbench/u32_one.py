"""Two fs_sort_keys_u32 calls on 2^28 uniform keys (for ncu launch lists)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import datagen
import paper_2605_10390_b200 as fs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
k = torch.empty(n, dtype=torch.uint32, device="cuda")
datagen.gen_u32_device(k.data_ptr(), n, seed=0, stream=torch.cuda.current_stream().cuda_stream)
out = torch.empty_like(k)
for _ in range(2):
    fs.sort_keys(k, out=out)
torch.cuda.synchronize()
