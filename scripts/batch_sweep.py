"""Batch-size sweep of the out-of-core path (the analog
of the paper's Batch Size Selection study):
fs_sort_keys_u16_host on c2's 2^28 uint16 keys from pinned host memory to pinned
host memory, one reused histogram, for batch sizes 2^18 .. 2^27 keys.  Prints
one JSON line per batch size (median of 5 sorts, CUDA events bracketing the
call on its stream; every output checked against the oracle once).

    python scripts/batch_sweep.py > profiles/r01c/batch_sweep.jsonl
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_10390_b200 as fs  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
    keys = datagen.gen_u16("uniform", n, seed=0)
    want = oracle.sort_u16(keys)
    host_in = torch.from_numpy(keys).pin_memory()
    host_out = torch.empty(n, dtype=torch.uint16).pin_memory()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for lg in range(18, 28):
        batch = 1 << lg
        work = torch.empty(fs.sort_keys_u16_host_work_bytes(n, batch), dtype=torch.uint8, device=dev)
        fs.sort_keys_u16_host(host_in, host_out, batch=batch, device=dev, work=work)
        ok = bool(np.array_equal(host_out.numpy(), want))
        times = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fs.sort_keys_u16_host(host_in, host_out, batch=batch, device=dev, work=work, synchronize=False)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = statistics.median(times)
        print(json.dumps({"batch_keys": batch, "batches": -(-n // batch), "ms": round(ms, 3),
                          "gkeys_per_s": round(n / (ms * 1e-3) / 1e9, 3),
                          "host_bytes_per_direction_over_sort_GBps": round(2 * n / (ms * 1e-3) / 1e9, 2),
                          "device_work_bytes": work.numel(), "verified": ok}), flush=True)
        del work
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
