"""Freeze the seeded generators: sha256 of the first 1024 keys of every
distribution (seed 0) -> tests/golden/datagen_first1024.json.

Calls only datagen/ (the generator module); nothing here comes from the CUDA path
or the oracle.  Re-run only when the generator recipe changes on purpose (and say
why in the commit message)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402


def h(a):
    return hashlib.sha256(a.tobytes()).hexdigest()


def main():
    out = {"_about": "sha256 of the first 1024 generated keys (little-endian) per distribution, seed 0; "
                     "written by scripts/make_golden_datagen.py from datagen/ only"}
    for d in ["uniform", "zipf", "gauss", "const"]:
        a = datagen.gen_u16(d, 1024, seed=0, n_total=1 << 28)
        out[f"u16_{d}"] = {"sha256": h(a), "first8": a[:8].tolist()}
    a = datagen.gen_u16("sortedswap", 1 << 20, seed=0)
    out["u16_sortedswap_n2^20"] = {"sha256": h(a[:1024]), "first8": a[:8].tolist()}
    a = datagen.gen_u64(1024, seed=0)
    out["u64_uniform"] = {"sha256": h(a), "first4": [int(x) for x in a[:4]]}
    a = datagen.gen_u32(1024, seed=0)
    out["u32_uniform"] = {"sha256": h(a), "first4": [int(x) for x in a[:4]]}
    path = os.path.join(ROOT, "tests", "golden", "datagen_first1024.json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
