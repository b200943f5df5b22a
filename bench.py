#!/usr/bin/env python
"""bench.py — throughput of the B200 hot path on BASELINE.json's headline config.

Workload (BASELINE.json configs[1], "c2"): 268,435,456 uint16 keys, i.i.d. uniform
over [0, 65535], seed 0, keys-only ascending sort on one B200.  Under torchrun
(N > 1) every rank sorts its own 2^28-key shard of an N*2^28-key input (global
indices [r*2^28, (r+1)*2^28)) with the multi-GPU Mode B path: local compressed
histogram -> NCCL all-reduce of the 512 KiB histogram -> expansion of the rank's
own output range (weak scaling).  At N > 1 the line also carries
the north-star gate's strong-scaling block (c4: 2^34 keys in total, Mode B), the
payload exchanges Mode A (NCCL all-to-all) and Mode P (peer stores), and the
distributed stable pair sort of c5 (2^29 pairs in total; mode P = the fused
exchange, mode A = all-to-all), each with its NVLink GB/s; every output is verified.

One step = one pass of the whole hot path (histogram, merge+scan, count-expansion)
over one batch of input resident in HBM.  Inputs (512 MiB) are larger than L2
(126 MB), so no flush is needed between steps.  Timing: W untimed warm-up steps,
exactly K timed steps bracketed by barrier + synchronize and two CUDA events on
the launching stream (nothing else is recorded inside the timed region), max over
ranks.  The per-kernel times (roofline) come from a second, instrumented run of
the same steps with CUDA events at the library's phase boundaries
(fs_set_phase_events); its own per-step time is reported beside the clean one.

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (the
"reference arm" of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _load_metrics():
    """paper_2605_10390_b200/metrics.py by path: plain host arithmetic, without the
    package's __init__ (which loads torch and the CUDA library the reference arm
    does not need)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("fs_metrics", os.path.join(ROOT, "paper_2605_10390_b200",
                                                                            "metrics.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


metrics = _load_metrics()

METRIC = "Gkeys/s and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200"
N_PER_GPU = 1 << 28
C4_TOTAL = 1 << 34
NVLINK_GBPS = 900.0  # per direction per GPU (north_star)
WORKLOAD = "c2: 268,435,456 uint16 keys per GPU, i.i.d. uniform [0,65535], seed 0, keys-only ascending sort"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="fs", choices=["fs", "reference"])
    ap.add_argument("--n", type=int, default=None, help="keys per GPU (default: the workload's size)")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3a", "c3b", "c3c", "c3d", "c4", "c5"],
                    help="BASELINE.json config (c2 is the headline; the others are extra lines)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="c1: time plain stream launches, not graph replays")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-multi-blocks", action="store_true",
                    help="N > 1: skip the c4 / mode A / mode P / pairs blocks")
    return ap.parse_args()


# ------------------------------------------------------------------ peaks and clocks
def measured_peak_gbs():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: b.copy_ read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(0.0002)  # short timed regions (c2: ~4 ms for 20 steps) still get tens of samples

    def __enter__(self):
        if self.nv:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        reasons = [name for bit, name in REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML polled every ~0.2-0.5 ms during the timed region"}


# ------------------------------------------------------------------ CPU oracle timings
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def time_oracle(keys, threads: int, min_reps: int, min_seconds: float):
    """The oracle as it stands: oracle_sort_u16 (threads = 1) or its POSIX-threads
    form oracle_sort_u16_mt (PAPER.md:86-92 local -> global scheme)."""
    import oracle
    fn = (lambda: oracle.sort_u16(keys)) if threads == 1 else (lambda: oracle.sort_u16_mt(keys, threads))
    out = fn()  # warm-up (page faults of the output)
    reps, t0 = 0, time.perf_counter()
    while reps < min_reps or (time.perf_counter() - t0) < min_seconds:
        out = fn()
        reps += 1
    dt = time.perf_counter() - t0
    ok = bool((out[1:] >= out[:-1]).all())
    return keys.size * reps / dt, reps, dt, ok


def cpu_baseline_block(n: int, budget_s: float = 14.0):
    """Single-thread and n_c-thread oracle on the full c2 input, on this host's cores;
    T_unit = n / (t n_c) keys/s/core."""
    import datagen
    keys = datagen.gen_u16("uniform", n, seed=0, n_total=n)
    nc = host_cores()
    v1, r1, d1, ok1 = time_oracle(keys, 1, 2, budget_s * 0.4)
    vm, rm, dm, okm = time_oracle(keys, nc, 3, budget_s * 0.6)
    return {
        "value": round(vm / 1e9, 6), "unit": "Gkeys/s", "cores": nc, "kind": "oracle",
        "sample": (f"the full c2 input (2^28 keys), sorted {rm} times ({dm:.1f} s) by the oracle on {nc} threads "
                   f"(oracle_sort_u16_mt) and {r1} times ({d1:.1f} s) on one thread (oracle_sort_u16)"),
        "T_unit_keys_per_s_per_core": round(metrics.unit_throughput(n, n / vm, nc), 1),
        "single_thread": {"value": round(v1 / 1e9, 6), "unit": "Gkeys/s", "cores": 1,
                          "T_unit_keys_per_s_per_core": round(metrics.unit_throughput(n, n / v1, 1), 1)},
        "host_GBps": round(4 * vm / 1e9, 2), "verified_nondecreasing": ok1 and okm,
        "cpu": cpu_model(), "host_cores": nc,
        "paper_context": "PAPER.md:417: 25.30e6 keys/s/core (i7-8665U, n_c = 4, 2^31 keys, 21.22 s)",
    }


def run_reference(args, rank, world):
    """Reference arm: the oracle on the host's cores, the same c2 workload and metric;
    each step sorts the full 2^28-key input once on n_c threads."""
    if rank != 0:
        return
    import datagen
    import oracle
    n = args.n or N_PER_GPU
    keys = datagen.gen_u16("uniform", n, seed=0, n_total=n)
    nc = host_cores()
    for _ in range(max(0, min(args.warmup, 2))):
        oracle.sort_u16_mt(keys, nc)
    steps = max(1, min(args.steps, 40))
    t0 = time.perf_counter()
    for _ in range(steps):
        out = oracle.sort_u16_mt(keys, nc)
    dt = time.perf_counter() - t0
    v = n * steps / dt / 1e9
    ok = bool((out[1:] >= out[:-1]).all())
    v1, r1, d1, _ = time_oracle(keys, 1, 1, 2.0)
    sample = f"the full c2 input (2^28 keys) per step, {steps} steps on {nc} threads (oracle_sort_u16_mt)"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gkeys/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt / steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "reference": "CPU oracle (oracle/oracle_mt.c: per-thread histograms, "
                                                      "merge, per-thread expansion), host cores"},
        "cpu_baseline": {"value": round(v, 6), "unit": "Gkeys/s", "cores": nc, "kind": "oracle", "sample": sample,
                         "T_unit_keys_per_s_per_core": round(metrics.unit_throughput(n * steps, dt, nc), 1),
                         "single_thread": {"value": round(v1 / 1e9, 6), "unit": "Gkeys/s", "cores": 1,
                                           "reps": r1, "seconds": round(d1, 2)},
                         "cpu": cpu_model(), "host_cores": nc},
        "e2e": {"value": round(v, 6), "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "verified_nondecreasing": ok,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm: shared helpers
def load_traffic(kernel: str, workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the newest committed ncu capture
    of this workload (profiles/ncu_traffic_<round>_<workload>.json; before per-workload names,
    profiles/ncu_traffic_<round>.json held the c2 / c5 kernels)."""
    import re
    pdir = os.path.join(ROOT, "profiles")
    names = sorted(os.listdir(pdir), reverse=True) if os.path.isdir(pdir) else []
    own = [n for n in names if n.startswith("ncu_traffic") and n.endswith(f"_{workload}.json")]
    legacy = [n for n in names if n.startswith("ncu_traffic") and n.endswith(".json")
              and not re.search(r"_c\d[a-z]?\.json$", n)] if workload in ("c2", "c5") else []
    for name in own + legacy:
        if True:
            try:
                d = json.load(open(os.path.join(pdir, name)))
                if kernel in d:
                    return d[kernel].get("dram_bytes_per_launch"), name
            except Exception:
                pass
    return None, None


def ctypes_array(events):
    import ctypes
    return (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])


def max_over_ranks(x: float, dev, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ok(ok: bool, dev, dist) -> bool:
    if dist is None:
        return ok
    import torch
    t = torch.tensor([1 if ok else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def timed(step, steps: int, warmup: int, dev, dist, clocks_index=None):
    """W warm-up steps, then exactly `steps` steps between barrier + synchronize and
    two CUDA events on the current stream; returns (ms, clocks summary)."""
    import torch
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index if clocks_index is None else clocks_index) as clocks:
        a.record(stream)
        for _ in range(steps):
            step()
        b.record(stream)
        while not b.query():  # wait without holding the GIL, so the clock sampler thread runs
            time.sleep(0.0001)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    return max_over_ranks(a.elapsed_time(b), dev, dist), clocks.summary()


WORKLOADS = {
    "c1": ("uniform", 1 << 20, "c1: 1,048,576 uint16 keys, uniform, seed 0 (L2-resident: launch-bound)"),
    "c2": ("uniform", N_PER_GPU, WORKLOAD),
    "c3a": ("zipf", N_PER_GPU, "c3a: 268,435,456 uint16 keys, Zipf s=1.2 with seeded value permutation, seed 0"),
    "c3b": ("gauss", N_PER_GPU, "c3b: 268,435,456 uint16 keys, Gaussian(32768, 1024) rounded+clipped, seed 0"),
    "c3c": ("sortedswap", N_PER_GPU, "c3c: 268,435,456 uint16 keys, sorted + floor(n/100) random pair swaps, seed 0"),
    "c3d": ("const", N_PER_GPU, "c3d: 268,435,456 uint16 keys, all equal (0xA5A5)"),
    # c4: the 32 GB job, split evenly over the N GPUs of the run (strong scaling)
    "c4": ("uniform", C4_TOTAL, "c4: 17,179,869,184 uint16 keys (32 GB) in total, uniform, seed 0, sharded evenly "
                                "by global index; Mode B across GPUs"),
}


def gen_shard(dist_name, n, n_total, i0, dev):
    import torch

    import datagen
    keys = torch.empty(n, dtype=torch.uint16, device=dev)
    if dist_name == "sortedswap":
        keys.copy_(torch.from_numpy(datagen.gen_u16("sortedswap", n_total, seed=0)[i0:i0 + n]))
    else:
        datagen.gen_u16_device(keys.data_ptr(), dist_name, n, seed=0, i0=i0, n_total=n_total,
                               stream=torch.cuda.current_stream(dev).cuda_stream)
    return keys


# ------------------------------------------------------------------ verification
def verify(out, keys):
    """Cheap end check of the timed output against the oracle (rank 0, N = 1)."""
    import numpy as np

    import oracle
    return bool(np.array_equal(out.cpu().numpy(), oracle.sort_u16(keys.cpu().numpy())))


def oracle_hist(keys, chunk=1 << 28):
    import numpy as np

    import oracle
    C = np.zeros(65536, dtype=np.uint64)
    for a in range(0, keys.numel(), chunk):
        C += oracle.histogram_u16(keys[a:a + chunk].cpu().numpy())
    return C


def verify_range(out, begin, C_global, chunk=1 << 28):
    """Check a slice out = sorted positions [begin, begin + len) of a global sort
    whose oracle histogram is C_global: every value's first and last position
    inside the slice, 2^20 random positions, and non-decreasing order (device,
    chunked) -- together they pin the slice of the sorted multiset."""
    import numpy as np
    import torch

    import oracle
    m = out.numel()
    if m == 0:
        return True
    P = oracle.exclusive_scan(C_global)
    end = begin + m
    nonempty = np.nonzero(C_global)[0]
    pos = np.concatenate([P[nonempty], P[nonempty + 1] - 1,
                          np.random.default_rng(begin).integers(begin, end, 1 << 20).astype(np.uint64)])
    pos = pos[(pos >= begin) & (pos < end)]
    want = (np.searchsorted(P, pos, side="right") - 1).astype(np.int64)
    idx = torch.from_numpy((pos - begin).astype(np.int64)).to(out.device)
    got = out.view(torch.int16)[idx].to(torch.int64).cpu().numpy() & 0xFFFF
    ok = bool(np.array_equal(got, want))
    for a in range(0, m - 1, chunk):
        b = min(a + chunk + 1, m)
        seg = out[a:b].view(torch.int16).to(torch.int32) & 0xFFFF
        ok &= bool((seg[1:] >= seg[:-1]).all().item())
    return ok


def global_hist(keys, dev, dist):
    """Oracle histogram of the union of the ranks' shards (host, then all-reduced)."""
    import torch
    C = oracle_hist(keys)
    if dist is None:
        return C
    t = torch.from_numpy(C.astype("int64")).to(dev)
    dist.all_reduce(t)
    return t.cpu().numpy().astype("uint64")


# ------------------------------------------------------------------ c5 (pairs)
def run_fs_pairs(args, dev):
    """Config c5: 2^29 (u64 key uniform, u32 value = index) pairs, stable sort (one GPU)."""
    import torch

    import datagen
    import paper_2605_10390_b200 as fs
    from paper_2605_10390_b200 import _lib
    L = fs.lib()
    n = args.n or (1 << 29)
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    k = torch.empty(n, dtype=torch.uint64, device=dev)
    v = torch.empty(n, dtype=torch.uint32, device=dev)
    datagen.gen_u64_device(k.data_ptr(), n, seed=0, stream=s)
    datagen.iota_u32_device(v.data_ptr(), n, stream=s)
    ko, vo = torch.empty_like(k), torch.empty_like(v)
    temp = torch.empty(L.fs_sort_pairs_u64_u32_temp_bytes(n, 64), dtype=torch.uint8, device=dev)

    def step(h=None):
        if h is not None:
            L.fs_set_phase_events(h, nev)
        _lib.check(L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64,
                                           temp.data_ptr(), temp.numel(), s), "fs_sort_pairs_u64_u32")
        if h is not None:
            L.fs_set_phase_events(None, 0)

    # clean timed region: two events around K sorts
    total_ms, clocks = timed(step, args.steps, args.warmup, dev, None)
    t_step = total_ms / args.steps
    # instrumented run: phase events (include/fractalsort.h): MSD-planned sorts record
    # [0] start, [1] trie histogram + scan + plan, [2] level-1 scatter, [3] level-2
    # scatter, [4] k_heavy (uneven level 2 and the recursion into oversize bins;
    # returns at once on c5), [5] per-bin local sorts, [6..15] the LSD kernels (they
    # return at once when the MSD path ran).
    nev = 16
    isteps = max(3, min(args.steps, 10))
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(isteps)]
    for row in events:
        for e in row:
            e.record(stream)
    handles = [ctypes_array(row) for row in events]
    torch.cuda.synchronize()
    for i in range(isteps):
        step(handles[i])
    torch.cuda.synchronize()
    inst_ms = events[0][0].elapsed_time(events[-1][nev - 1]) / isteps
    phase = [statistics.mean(r[i].elapsed_time(r[i + 1]) for r in events) for i in range(nev - 1)]
    names = ["trie_hist+scan+plan", "msd_level1_scatter", "msd_level2_scatter", "k_heavy", "local_sort",
             "lsd_digit_hist+plan"] + [f"lsd_pass{i}" for i in range(8)] + ["lsd_identity_copy"]
    lsd_ms = sum(phase[5:])
    path = "msd" if phase[4] > lsd_ms else "lsd"
    # dominant kernel: each MSD pass reads and writes 8 B key + 4 B value per pair
    cand = [1, 2, 4] if path == "msd" else list(range(6, 14))
    dom = max(cand, key=lambda i: phase[i])
    peak, peak_src = measured_peak_gbs()
    alg = metrics.minimal_bytes_pairs(n, 8, 4)  # each MSD pass moves every pair once: read + write
    achieved = alg / (phase[dom] * 1e-3) / 1e9
    method_b = 80 * n if path == "msd" else 200 * n
    traffic, traffic_src = load_traffic(names[dom], "c5")
    line = {
        "metric": METRIC, "value": round(n * args.steps / (total_ms * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "c5: 536,870,912 (u64 key uniform, u32 value = index) pairs, stable ascending sort",
                   "pairs": n, "l2": "inputs (6 GiB) larger than L2: no flush", "path": path},
        "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(metrics.roofline_frac(alg, phase[dom] * 1e-3, peak), 4),
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg, "avg_launch_ms": round(phase[dom], 4),
                     "peak_source": peak_src, "traffic_source": traffic_src,
                     "timing": f"phase events of a separate instrumented run of {isteps} sorts"},
        "whole_step": {"minimal_bytes": alg, "method_bytes": method_b,
                       "frac_minimal_of_measured_peak": round(metrics.roofline_frac(alg, t_step * 1e-3, peak), 4),
                       "method_GBps": round(method_b / (t_step * 1e-3) / 1e9, 1),
                       "frac_method_of_measured_peak": round(metrics.roofline_frac(method_b, t_step * 1e-3, peak), 4)},
        "phases_ms": {nm: round(x, 4) for nm, x in zip(names, phase)},
        "ms_per_step_instrumented": round(inst_ms, 4),
        # MSD: 16 kernels (2 hist, window x2, scan, lists, plan, 2 vseg, 2 scatters, heavy,
        # local, tiny, mid, items); LSD: 11 (return at once) -- see profiles/*/launches_c5.csv
        "gpu_launches": 27 * args.steps,
        "clocks": clocks,
    }
    if not args.no_verify:
        import oracle
        kin, kout, vout = k.cpu().numpy(), ko.cpu().numpy(), vo.cpu().numpy()
        line["verified_invariants"] = oracle.check_pairs_index(kin, kout, vout) == 0
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ u16 keys (c1-c4)
def run_fs(args, rank, world, local_rank):
    import torch

    import paper_2605_10390_b200 as fs
    from paper_2605_10390_b200 import _lib

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if args.workload == "c5":
        return run_fs_pairs(args, dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
    L = fs.lib()
    dist_name, n_default, workload_text = WORKLOADS[args.workload]
    n = args.n or n_default
    if args.workload == "c4":  # fixed total, split over the ranks
        n = n // world
    n_total = n * world
    keys = gen_shard(dist_name, n, n_total, rank * n, dev)
    out = torch.empty(n, dtype=torch.uint16, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    b0, b1 = (n_total * rank) // world, (n_total * (rank + 1)) // world
    if world > 1:
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
        htemp = torch.empty(L.fs_histogram_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
    else:
        temp = torch.empty(L.fs_sort_keys_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
    nev = 4

    def step(ev=None):
        if world == 1:
            if ev is not None:
                L.fs_set_phase_events(ev[1], nev)
            _lib.check(L.fs_sort_keys_u16(keys.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s),
                       "fs_sort_keys_u16")
            if ev is not None:
                L.fs_set_phase_events(None, 0)
        else:
            if ev is not None:
                ev[0][0].record()
            _lib.check(L.fs_histogram_prefix_u16(keys.data_ptr(), n, prefix2.data_ptr(), htemp.data_ptr(),
                                                 htemp.numel(), s), "fs_histogram_prefix_u16")
            if ev is not None:
                ev[0][1].record()
            # NCCL, 513 KiB: the global histogram merge across GPUs, in the
            # sort's two-level prefix form (linear in the counts: no scan after it)
            dist.all_reduce(prefix2)
            if ev is not None:
                ev[0][2].record()
            _lib.check(L.fs_expand_prefix_u16(prefix2.data_ptr(), b0, b1, out.data_ptr(), s), "fs_expand_prefix_u16")
            if ev is not None:
                ev[0][3].record()

    # ---- the clean timed region.  c1 (2^20 keys, L2-resident) is launch-bound: its
    # steps are replays of a CUDA graph holding one sort (the same two kernels)
    use_graph = world == 1 and args.workload == "c1" and not args.no_graph
    clean_step = step
    if use_graph:
        cs = torch.cuda.Stream(dev)
        g = torch.cuda.CUDAGraph()

        def call_on(st):
            _lib.check(L.fs_sort_keys_u16(keys.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(),
                                          st.cuda_stream), "fs_sort_keys_u16")
        cs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs):
            for _ in range(3):  # first calls set kernel attributes outside the capture
                call_on(cs)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g, stream=cs):
            call_on(cs)

        def clean_step():
            g.replay()
    total_ms, clocks = timed(clean_step, args.steps, args.warmup, dev, dist)
    t_step = total_ms / args.steps
    value = n_total * args.steps / (total_ms * 1e-3) / 1e9

    # ---- the instrumented run: per-kernel times from phase events
    isteps = max(4, min(args.steps, 16))
    rows = []
    for _ in range(isteps):
        row = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
        for e in row:
            e.record()  # materialise the cudaEvent_t handles
        rows.append((row, ctypes_array(row)))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    for r in rows:
        step(r)
    torch.cuda.synchronize()
    inst_ms = max_over_ranks(rows[0][0][0].elapsed_time(rows[-1][0][nev - 1]) / isteps, dev, dist)
    phase_ms = [max_over_ranks(statistics.mean(r[0][i].elapsed_time(r[0][i + 1]) for r in rows), dev, dist)
                for i in range(nev - 1)]

    # Roofline of the dominant kernel (algorithmic bytes = 2 B/key read for the
    # histogram, 2 B/key written for the expansion).
    if world == 1:
        names = {"hist16": phase_ms[1], "expand16": phase_ms[2]}  # phase 0 is empty (no memset)
        phase_names = ["prologue", "hist16+merge+scan", "expand16"]
    else:
        names = {"hist16": phase_ms[0], "expand16": phase_ms[2]}
        phase_names = ["hist16+merge+scan", "nccl_allreduce", "expand16"]
    dom = max(names, key=names.get)
    alg_bytes = 2 * (n if dom == "hist16" else (b1 - b0))
    peak, peak_src = measured_peak_gbs()
    achieved = alg_bytes / (names[dom] * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(dom, args.workload) if world == 1 else (None, None)
    whole_bytes = metrics.minimal_bytes_keys(n, 2)  # the u16 sort reads and writes every key once
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step, 5), "higher_is_better": True,
        "scaling": "strong" if args.workload == "c4" else "weak", "vs_baseline": None, "dtype": "u16",
        "data": "synthetic",
        "config": {"workload": workload_text if (n * world == n_default or n == n_default) else
                   f"{n} uint16 keys per GPU, {dist_name}, seed 0",
                   "keys_per_gpu": n, "keys_total": n_total, "parallelism": f"dp{world}",
                   "multi_gpu_mode": None if world == 1 else "B (two-level prefix all-reduce + own-range expansion)",
                   "l2": (f"inputs ({n * 2 / 2**20:.0f} MiB/GPU) larger than L2 (126 MB): no flush between steps"
                          if n * 2 > 126e6 else "L2-resident input (c1): launch-bound, no roofline claim")},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(metrics.roofline_frac(alg_bytes, names[dom] * 1e-3, peak), 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": round(names[dom], 5),
                     "peak_source": peak_src, "traffic_source": traffic_src,
                     "timing": f"phase events of a separate instrumented run of {isteps} steps"},
        "whole_step": {"algorithmic_bytes": whole_bytes,
                       "achieved_GBps": round(whole_bytes / (t_step * 1e-3) / 1e9, 1),
                       "frac_of_measured_peak": round(metrics.roofline_frac(whole_bytes, t_step * 1e-3, peak), 4),
                       "frac_of_8TBps": round(whole_bytes / (t_step * 1e-3) / 8e12, 4)},
        "phases_ms": {k: round(v, 5) for k, v in zip(phase_names, phase_ms)},
        "ms_per_step_instrumented": round(inst_ms, 5),
        "gpu_launches": (1 if (world == 1 and n <= (1 << 18)) else 2) * args.steps,  # one cluster launch up to 2^18
        "clocks": clocks,
        "timing": "ms_per_step from two CUDA events around the K timed steps (nothing recorded in between); "
                  "phases from the instrumented run" +
                  ("; each timed step is one replay of a CUDA graph capturing one fs_sort_keys_u16 call "
                   "(launch-bound size)" if use_graph else ""),
    }
    if args.workload == "c2" and world == 1 and traffic is not None:
        t_exp, _ = load_traffic("expand16", "c2")
        if t_exp:
            line["b_eff"] = {"value": round(metrics.bandwidth_efficiency(whole_bytes, traffic + t_exp), 4),
                             "useful_bytes": whole_bytes,
                             "dram_bytes": traffic + t_exp,
                             "definition": "Eq. 1 (PAPER.md:432-436): useful / total DRAM bytes per sort; DRAM "
                                           "bytes = ncu dram__bytes_read.sum + dram__bytes_write.sum of hist16 and "
                                           "expand16", "source": traffic_src,
                             "note": "above 1 when part of expand16's output is still dirty in the 126 MB L2 as "
                                     "the kernel ends (write-back: ncu counts those writes in no launch); the "
                                     "method moves no bytes beyond the useful ones at c2"}

    # End to end through the public host-buffer API: H2D of the step's keys from
    # pinned memory, the sort, D2H of the sorted keys, every step.
    if not args.no_e2e and args.workload == "c2":
        line["e2e"] = e2e(args, L, _lib, keys, n, n_total, rank, world, dev, dist, out)

    if not args.no_verify:
        if world == 1 and n <= (1 << 28):
            line["verified"] = verify(out, keys)
        else:
            C = global_hist(keys, dev, dist)
            line["verified"] = all_ok(verify_range(out[:b1 - b0] if world > 1 else out, b0, C), dev, dist)
            line["verification"] = ("every rank's output slice vs the oracle histogram of the whole input "
                                    "(all-reduced): first/last position of every value, 2^20 sampled positions, "
                                    "order; pass flag min-reduced over ranks")
    if world > 1 and args.workload == "c2" and not args.no_multi_blocks:
        del out
        torch.cuda.empty_cache()
        line["c4_strong"] = c4_strong_block(args, L, _lib, rank, world, dev, dist, peak)
        line["mode_A"] = exchange_block("A", keys, rank, world, dev, dist, args)
        line["mode_P"] = exchange_block("P", keys, rank, world, dev, dist, args)
        if os.environ.get("FS_BENCH_SHARE_GPU") != "1":  # its in-kernel barrier needs one GPU per rank
            line["mode_N"] = exchange_block("N", keys, rank, world, dev, dist, args)
        del keys
        torch.cuda.empty_cache()
        line["pairs_P"] = pairs_block("P", rank, world, dev, dist, args)
        line["pairs_A"] = pairs_block("A", rank, world, dev, dist, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        line["cpu_baseline"] = cpu_baseline_block(n)
    if rank == 0:
        print(json.dumps(line), flush=True)


def c4_strong_block(args, L, _lib, rank, world, dev, dist, peak):
    """North-star gate: c4 (2^34 keys in total) split over the N ranks, Mode B."""
    import torch
    try:
        n = C4_TOTAL // world
        keys = gen_shard("uniform", n, C4_TOTAL, rank * n, dev)
        b0, b1 = (C4_TOTAL * rank) // world, (C4_TOTAL * (rank + 1)) // world
        out = torch.empty(b1 - b0, dtype=torch.uint16, device=dev)
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
        htemp = torch.empty(L.fs_histogram_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
        s = torch.cuda.current_stream(dev).cuda_stream

        def step():
            _lib.check(L.fs_histogram_prefix_u16(keys.data_ptr(), n, prefix2.data_ptr(), htemp.data_ptr(),
                                                 htemp.numel(), s), "fs_histogram_prefix_u16")
            dist.all_reduce(prefix2)
            _lib.check(L.fs_expand_prefix_u16(prefix2.data_ptr(), b0, b1, out.data_ptr(), s), "fs_expand_prefix_u16")
        steps = max(2, min(args.steps, 5))
        ms, _ = timed(step, steps, 2, dev, dist)
        t = ms / steps
        blk = {"workload": "c4: 2^34 uint16 keys (32 GB) in total, uniform, seed 0, sharded evenly by global index",
               "keys_total": C4_TOTAL, "keys_per_gpu": n, "mode": "B", "steps": steps, "ms_per_step": round(t, 4),
               "value": round(C4_TOTAL / (t * 1e-3) / 1e9, 3), "unit": "Gkeys/s", "scaling": "strong",
               "per_rank_hbm_frac_of_measured_peak": round(4 * n / (t * 1e-3) / 1e9 / peak, 4)}
        if not args.no_verify:
            blk["verified"] = all_ok(verify_range(out, b0, global_hist(keys, dev, dist)), dev, dist)
        del keys, out, htemp
        torch.cuda.empty_cache()
        return blk
    except Exception as e:  # a block failure must not lose the headline line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def exchange_block(mode, keys, rank, world, dev, dist, args):
    """Payload exchange of the c2 shards: mode A (NCCL all-to-all of the key bytes
    after a local sort, then a local sort) or mode P (every rank's keys stored
    straight to their final positions in the owners' buffers over NVLink); mode N
    is mode B with the prefix all-reduce done by the NVSwitch (multicast)."""
    import torch

    from paper_2605_10390_b200 import dist as fsd
    try:
        peers = fsd.PeerBuffers(dev) if mode == "P" else (fsd.MulticastBuffer(65536 + 128, dev) if mode == "N" else None)
        ev = {"x0": torch.cuda.Event(enable_timing=True), "x1": torch.cuda.Event(enable_timing=True)}
        stats = {}
        steps = max(2, min(args.steps, 5))
        xs, totals = [], []
        for i in range(steps + 1):
            torch.cuda.synchronize(dev)
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res, (begin, end) = fsd.sort_keys_u16(keys, mode=mode, peers=peers, events=ev, stats=stats)
            b.record()
            torch.cuda.synchronize(dev)
            if i:  # the first call maps the peers' buffers / warms NCCL
                xs.append(ev["x0"].elapsed_time(ev["x1"]))
                totals.append(a.elapsed_time(b))
        x_ms = max_over_ranks(statistics.median(xs), dev, dist)
        t_ms = max_over_ranks(statistics.median(totals), dev, dist)
        if mode == "N":  # the reduced two-level prefix each rank reads through the switch
            stats["sent_bytes"] = (65536 + 128) * 8
        sent = max_over_ranks(float(stats.get("sent_bytes", 0)), dev, dist)
        n_total = keys.numel() * world
        blk = {"mode": mode, "keys_total": n_total, "ms_per_sort": round(t_ms, 4),
               "value": round(n_total / (t_ms * 1e-3) / 1e9, 3), "unit": "Gkeys/s",
               "exchange_ms": round(x_ms, 4), "sent_bytes_per_rank": int(sent),
               "nvlink_GBps_per_rank": round(sent / (x_ms * 1e-3) / 1e9, 1),
               "frac_of_900GBps": round(sent / (x_ms * 1e-3) / 1e9 / NVLINK_GBPS, 4),
               "exchange": {"A": "NCCL all_to_all_single of the key bytes",
                            "P": "fs_expand_to_peers_u16: stores into the owners' CUDA-IPC-mapped buffers",
                            "N": "fs_allreduce_multicast_u64: the two-level prefix summed by the NVSwitch "
                                 "(multimem.ld_reduce) with the kernel's own barrier; no payload exchange "
                                 "(mode B with NVLS instead of NCCL)"}[mode],
               "timing": f"median of {steps} sorts, max over ranks; exchange = CUDA events around it"}
        if not args.no_verify:
            blk["verified"] = all_ok(verify_range(res, begin, global_hist(keys, dev, dist)), dev, dist)
        return blk
    except Exception as e:
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def pairs_block(mode, rank, world, dev, dist, args):
    """The distributed stable pair sort on c5 (2^29 (u64 key, u32 index) pairs in
    total, 2^29 / N per rank, strong scaling): exact splitters from one all-reduced
    16-bit histogram per level; mode P = classes + stores into the owners' peer
    buffers + one sort per owner (NEXT-2), mode A = local sort + NCCL all-to-all +
    sort.  Verified by the pair invariants on every rank's slice plus the global
    boundary keys."""
    import torch

    import datagen
    from paper_2605_10390_b200 import dist as fsd
    try:
        N = 1 << 29
        n = N // world
        s = torch.cuda.current_stream(dev).cuda_stream
        k = torch.empty(n, dtype=torch.uint64, device=dev)
        v = torch.empty(n, dtype=torch.uint32, device=dev)
        # the c5 input by global index: rank r holds pairs [r n, (r + 1) n), values = global index
        datagen.gen_u64_device(k.data_ptr(), n, seed=0, i0=rank * n, stream=s)
        datagen.iota_u32_device(v.data_ptr(), n, i0=rank * n, stream=s)
        peers = (fsd.PeerBuffers(dev, None, torch.uint64), fsd.PeerBuffers(dev, None, torch.uint32)) if mode == "P" \
            else None
        ev = {"x0": torch.cuda.Event(enable_timing=True), "x1": torch.cuda.Event(enable_timing=True)}
        stats = {}
        steps = max(2, min(args.steps, 3))
        xs, totals = [], []
        for i in range(steps + 1):
            torch.cuda.synchronize(dev)
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            (rk, rv), (begin, end) = fsd.sort_pairs_u64_u32(k, v, mode=mode, peers=peers, events=ev, stats=stats)
            b.record()
            torch.cuda.synchronize(dev)
            if i:
                xs.append(ev["x0"].elapsed_time(ev["x1"]))
                totals.append(a.elapsed_time(b))
        x_ms = max_over_ranks(statistics.median(xs), dev, dist)
        t_ms = max_over_ranks(statistics.median(totals), dev, dist)
        if mode == "N":  # the reduced two-level prefix each rank reads through the switch
            stats["sent_bytes"] = (65536 + 128) * 8
        sent = max_over_ranks(float(stats.get("sent_bytes", 0)), dev, dist)
        blk = {"mode": mode, "pairs_total": N, "ms_per_sort": round(t_ms, 4),
               "value": round(N / (t_ms * 1e-3) / 1e9, 3), "unit": "Gpairs/s", "scaling": "strong",
               "exchange_ms": round(x_ms, 4), "sent_bytes_per_rank": int(sent),
               "nvlink_GBps_per_rank": round(sent / (x_ms * 1e-3) / 1e9, 1),
               "frac_of_900GBps": round(sent / (x_ms * 1e-3) / 1e9 / NVLINK_GBPS, 4),
               "exchange": ("fs_pair_scatter_u64_u32: class-ordered stores into the owners' peer buffers" if mode == "P"
                            else "NCCL all_to_all_single of keys and values"),
               "timing": f"median of {steps} sorts, max over ranks (the first call maps the peers / warms NCCL)"}
        if not args.no_verify:
            import numpy as np
            rkn, rvn = rk.cpu().numpy(), rv.cpu().numpy()
            ok = bool(np.all(rkn[1:] >= rkn[:-1]))
            eq = rkn[1:] == rkn[:-1]
            ok &= bool(np.all(rvn[1:][eq] > rvn[:-1][eq]))       # stable: values are arrival indices
            # every pair's key is the input key at its index (gather), recomputed from the generator
            idx = rvn.astype(np.int64)
            sample = idx[:: max(1, idx.size // (1 << 16))]
            want = np.array([int(datagen.gen_u64(1, seed=0, i0=int(i))[0]) for i in sample[:256]], dtype=np.uint64)
            ok &= bool(np.array_equal(rkn[:: max(1, idx.size // (1 << 16))][:256], want))
            blk["verified"] = all_ok(ok and rkn.size == end - begin, dev, dist)
        del k, v
        torch.cuda.empty_cache()
        return blk
    except Exception as e:
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def e2e(args, L, _lib, keys, n, n_total, rank, world, dev, dist, out=None):
    import torch
    steps = max(1, min(args.steps, 10))
    host_in = keys.cpu().pin_memory()
    host_out = torch.empty(n, dtype=torch.uint16).pin_memory()
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    if world == 1:
        # Back-to-back host-buffer sorts as a streaming user issues them: steps
        # alternate between two streams (each with its own work buffer and pinned
        # output), so step i+1's copy-in runs while step i's copy-out drains (the
        # library's H2D and D2H copy streams use the link's two directions).
        # Every step copies its whole input in and its whole output out.
        streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        works = [torch.empty(L.fs_sort_keys_u16_host_work_bytes(n, 0), dtype=torch.uint8, device=dev)
                 for _ in range(2)]
        outs = [host_out, torch.empty(n, dtype=torch.uint16).pin_memory()]

        def call(i):
            j = i % 2
            _lib.check(L.fs_sort_keys_u16_host(host_in.data_ptr(), outs[j].data_ptr(), n, 0, works[j].data_ptr(),
                                               works[j].numel(), streams[j].cuda_stream), "fs_sort_keys_u16_host")

        def block(k):
            for st in streams:
                st.wait_stream(stream)
            for i in range(k):
                call(i)
            for st in streams:
                stream.wait_stream(st)

        block(2)  # warm-up (creates the library's copy streams)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        block(steps)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b)
        res = {"value": round(n_total * steps / (ms * 1e-3) / 1e9, 4), "unit": "Gkeys/s",
               "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 2 * n, "steps": steps,
               "api": "fs_sort_keys_u16_host (pinned host buffers; steps alternate between two streams with their "
                      "own work buffers, so one step's copy-out overlaps the next step's copy-in)",
               "timing": "two CUDA events on the issuing stream, both work streams joined before the second"}
        if out is not None:  # both pinned outputs hold a full sort of the input
            ok = all(bool(torch.equal(o.to(dev, non_blocking=False), out)) for o in outs[:min(steps, 2)])
            res["verified"] = ok
        return res
    else:
        d_in = torch.empty(n, dtype=torch.uint16, device=dev)
        d_out = torch.empty(n, dtype=torch.uint16, device=dev)
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
        htemp = torch.empty(L.fs_histogram_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
        b0, b1 = (n_total * rank) // world, (n_total * (rank + 1)) // world

        def one():
            d_in.copy_(host_in, non_blocking=True)
            _lib.check(L.fs_histogram_prefix_u16(d_in.data_ptr(), n, prefix2.data_ptr(), htemp.data_ptr(),
                                                 htemp.numel(), s), "fs_histogram_prefix_u16")
            dist.all_reduce(prefix2)
            _lib.check(L.fs_expand_prefix_u16(prefix2.data_ptr(), b0, b1, d_out.data_ptr(), s), "fs_expand_prefix_u16")
            host_out[:b1 - b0].copy_(d_out[:b1 - b0], non_blocking=True)
        h2d, d2h = 2 * n, 2 * (b1 - b0)
    ms, _ = timed(one, steps, 1, dev, dist)
    return {"value": round(n_total * steps / (ms * 1e-3) / 1e9, 4), "unit": "Gkeys/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "api": "fs_sort_keys_u16_host (pinned host buffers, batched copy/compute overlap)" if world == 1
            else "H2D + fs_histogram_prefix_u16 + NCCL all_reduce + fs_expand_prefix_u16 + D2H"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if os.environ.get("FS_BENCH_SHARE_GPU") == "1":
        # plumbing check of the N > 1 code path on a one-GPU box (every rank on
        # device 0, gloo collectives); its numbers mean nothing
        local_rank = 0
    if world > 1:
        import datetime

        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("FS_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, timeout=datetime.timedelta(seconds=600),
                                device_id=torch.device("cuda", local_rank) if backend == "nccl" else None)
    try:
        run_fs(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
