"""Stress: N random wide sorts (tests/test_gpu_wide.py::_fuzz_shape shapes, sizes
log-uniform up to 8M) against the oracle; prints failures and a summary."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen, oracle
import paper_2605_10390_b200 as fs
src = open(os.path.join(ROOT, "tests/test_gpu_wide.py")).read()
ns = {}
exec("import numpy as np\nimport datagen\n" + src[src.index("def _fuzz_shape"):src.index("@pytest.mark.parametrize(\"case\", range(24))")], ns)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bad = 0
for case in range(N):
    rng = np.random.default_rng(90000 + case)
    n = int(np.exp(rng.uniform(0, np.log(8_000_000))))
    k, kb = ns["_fuzz_shape"](rng, n)
    v = datagen.iota_u32(n)
    ko, vo = fs.sort_pairs(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), key_bits=kb)
    ek, ev = oracle.sort_pairs_u64_u32(k, v, kb)
    okk = np.array_equal(ko.cpu().numpy(), ek) and np.array_equal(vo.cpu().numpy(), ev)
    k2 = fs.sort_keys(torch.from_numpy(k).cuda(), key_bits=kb).cpu().numpy()
    ok2 = np.array_equal(k2, ek)
    if not (okk and ok2):
        bad += 1
        print(f"FAIL case={case} n={n} kb={kb} pairs={okk} keys={ok2}", flush=True)
print(f"fuzz: {N - bad}/{N} cases bit-exact", flush=True)
