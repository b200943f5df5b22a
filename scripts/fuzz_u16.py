"""Stress: N random u16 sorts (sizes log-uniform up to 2^23, mixtures of uniform,
Zipf, constant runs, hot keys, sorted data; random misalignment) against the oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen, oracle
import paper_2605_10390_b200 as fs
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bad = 0
for case in range(N):
    rng = np.random.default_rng(70000 + case)
    n = int(np.exp(rng.uniform(0, np.log(8_400_000))))
    dist = str(rng.choice(["uniform", "zipf", "gauss", "sortedswap", "const"]))
    k = datagen.gen_u16(dist, n, seed=int(rng.integers(1 << 30)))
    if rng.random() < 0.3:  # a hot key
        sel = datagen.gen_u16("uniform", n, seed=case).astype(np.float64) / 65536 < rng.uniform(0.05, 0.7)
        k[sel] = np.uint16(int(rng.integers(65536)))
    off = int(rng.integers(0, 8))
    d = torch.from_numpy(np.concatenate([np.zeros(off, np.uint16), k])).cuda()[off:]
    out = fs.sort_keys(d).cpu().numpy()
    if not np.array_equal(out, oracle.sort_u16(k)):
        bad += 1
        print(f"FAIL case={case} n={n} dist={dist} off={off}", flush=True)
print(f"fuzz u16: {N - bad}/{N} cases bit-exact", flush=True)
