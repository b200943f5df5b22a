#!/usr/bin/env python
"""bench.py — throughput of the B200 hot path on BASELINE.json's headline config.

Workload (BASELINE.json configs[1], "c2"): 268,435,456 uint16 keys, i.i.d. uniform
over [0, 65535], seed 0, keys-only ascending sort on one B200.  Under torchrun
(N > 1) every rank sorts its own 2^28-key shard of an N*2^28-key input (global
indices [r*2^28, (r+1)*2^28)) with the multi-GPU Mode B path: local compressed
histogram -> NCCL all-reduce of the 512 KiB histogram -> scan -> expansion of the
rank's own output range (weak scaling).

One step = one pass of the whole hot path (histogram, merge+scan, count-expansion)
over one batch of input resident in HBM.  Inputs (512 MiB) are larger than L2
(126 MB), so no flush is needed between steps.  Timing: CUDA events recorded by
the library at its phase boundaries (fs_set_phase_events) on the launching
stream, W untimed warm-up steps, exactly K timed steps bracketed by barrier +
synchronize, max over ranks.

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (the
"reference arm" of this tier) on a bounded sample of the same workload.
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

METRIC = "Gkeys/s and achieved HBM GB/s (% of roofline) at 1/2/4/8 B200"
PHASE_EVERY = 8  # phase events recorded on every 8th timed step
N_PER_GPU = 1 << 28
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
    ap.add_argument("--no-verify", action="store_true")
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
            time.sleep(0.002)

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
                "source": "NVML polled every ~2 ms during the timed region"}


# ------------------------------------------------------------------ reference arm (CPU oracle)
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


def time_oracle(n_sample: int, steps: int, warmup: int, min_seconds: float = 0.0):
    """The oracle as it stands (single-threaded C counting sort) on a bounded sample."""
    import numpy as np  # noqa: F401

    import datagen
    import oracle
    keys = datagen.gen_u16("uniform", n_sample, seed=0, n_total=N_PER_GPU)
    for _ in range(warmup):
        oracle.sort_u16(keys)
    reps, t0 = 0, time.perf_counter()
    while reps < steps or (time.perf_counter() - t0) < min_seconds:
        out = oracle.sort_u16(keys)
        reps += 1
    dt = time.perf_counter() - t0
    ok = bool((out[1:] >= out[:-1]).all())
    return n_sample * reps / dt / 1e9, reps, dt, ok


def run_reference(args, rank, world):
    if rank != 0:
        return
    n_sample = 1 << 26
    v, reps, dt, ok = time_oracle(n_sample, args.steps, args.warmup)
    sample = f"first 2^26 keys of the c2 input per step (1/4 of the 2^28-key workload), {reps} steps"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gkeys/s", "n_gpus": args.gpus,
        "steps": reps, "warmup": args.warmup, "ms_per_step": round(dt / reps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "reference": "CPU oracle (oracle/oracle.c counting sort), single thread"},
        "cpu_baseline": {"value": round(v, 6), "unit": "Gkeys/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model(), "host_cores": host_cores()},
        "e2e": {"value": round(v, 6), "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "verified_nondecreasing": ok,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def load_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_traffic") and name.endswith(".json"):
            try:
                d = json.load(open(os.path.join(ROOT, "profiles", name)))
                if kernel in d:
                    return d[kernel].get("dram_bytes_per_launch"), name
            except Exception:
                pass
    return None, None


WORKLOADS = {
    "c1": ("uniform", 1 << 20, "c1: 1,048,576 uint16 keys, uniform, seed 0 (L2-resident: launch-bound)"),
    "c2": ("uniform", N_PER_GPU, WORKLOAD),
    "c3a": ("zipf", N_PER_GPU, "c3a: 268,435,456 uint16 keys, Zipf s=1.2 with seeded value permutation, seed 0"),
    "c3b": ("gauss", N_PER_GPU, "c3b: 268,435,456 uint16 keys, Gaussian(32768, 1024) rounded+clipped, seed 0"),
    "c3c": ("sortedswap", N_PER_GPU, "c3c: 268,435,456 uint16 keys, sorted + floor(n/100) random pair swaps, seed 0"),
    "c3d": ("const", N_PER_GPU, "c3d: 268,435,456 uint16 keys, all equal (0xA5A5)"),
    # c4: the 32 GB job, split evenly over the N GPUs of the run (strong scaling)
    "c4": ("uniform", 1 << 34, "c4: 17,179,869,184 uint16 keys (32 GB) in total, uniform, seed 0, sharded evenly "
                               "by global index; Mode B across GPUs"),
}


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
    # phase events (include/fractalsort.h): MSD-planned sorts record [0] start,
    # [1] trie histogram + scan + plan, [2] level-1 scatter, [3] level-2 scatter,
    # [4] k_heavy (uneven level 2 and the recursion into oversize bins; returns
    # at once on c5), [5] per-bin local sorts, [6..15] the LSD kernels (they
    # return at once when the MSD path ran).
    nev = 16
    steps = args.steps
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(steps)]
    for row in events:
        for e in row:
            e.record(stream)
    handles = [ctypes_array(row) for row in events]
    torch.cuda.synchronize()

    def step(h=None):
        if h is not None:
            L.fs_set_phase_events(h, nev)
        _lib.check(L.fs_sort_pairs_u64_u32(k.data_ptr(), v.data_ptr(), ko.data_ptr(), vo.data_ptr(), n, 64,
                                           temp.data_ptr(), temp.numel(), s), "fs_sort_pairs_u64_u32")
        if h is not None:
            L.fs_set_phase_events(None, 0)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        for i in range(steps):
            step(handles[i])
        torch.cuda.synchronize()
    total_ms = events[0][0].elapsed_time(events[-1][nev - 1])
    phase = [statistics.mean(r[i].elapsed_time(r[i + 1]) for r in events) for i in range(nev - 1)]
    names = ["trie_hist+scan+plan", "msd_level1_scatter", "msd_level2_scatter", "k_heavy", "local_sort",
             "lsd_digit_hist+plan"] + [f"lsd_pass{i}" for i in range(8)] + ["lsd_identity_copy"]
    lsd_ms = sum(phase[5:])
    path = "msd" if phase[4] > lsd_ms else "lsd"
    # dominant kernel: each MSD pass reads and writes 8 B key + 4 B value per pair
    cand = [1, 2, 4] if path == "msd" else list(range(6, 14))
    dom = max(cand, key=lambda i: phase[i])
    peak, peak_src = measured_peak_gbs()
    alg = 24 * n
    achieved = alg / (phase[dom] * 1e-3) / 1e9
    t_step = total_ms / steps
    method_b = 80 * n if path == "msd" else 200 * n
    traffic, traffic_src = load_traffic(names[dom])
    line = {
        "metric": METRIC, "value": round(n * steps / (total_ms * 1e-3) / 1e9, 3), "unit": "Gkeys/s", "n_gpus": 1,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "c5: 536,870,912 (u64 key uniform, u32 value = index) pairs, stable ascending sort",
                   "pairs": n, "l2": "inputs (6 GiB) larger than L2: no flush", "path": path},
        "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg, "avg_launch_ms": round(phase[dom], 4),
                     "peak_source": peak_src, "traffic_source": traffic_src},
        "whole_step": {"minimal_bytes": 24 * n, "method_bytes": method_b,
                       "frac_minimal_of_measured_peak": round(24 * n / (t_step * 1e-3) / 1e9 / peak, 4),
                       "method_GBps": round(method_b / (t_step * 1e-3) / 1e9, 1),
                       "frac_method_of_measured_peak": round(method_b / (t_step * 1e-3) / 1e9 / peak, 4)},
        "phases_ms": {nm: round(x, 4) for nm, x in zip(names, phase)},
        # MSD: 16 kernels (2 hist, window x2, scan, lists, plan, 2 vseg, 2 scatters, heavy,
        # local, tiny, mid, items); LSD: 11 (return at once) -- see profiles/*/launches_c5.csv
        "gpu_launches": 27 * steps,
        "clocks": clocks.summary(),
    }
    if not args.no_verify:
        import oracle
        kin, kout, vout = k.cpu().numpy(), ko.cpu().numpy(), vo.cpu().numpy()
        line["verified_invariants"] = oracle.check_pairs_index(kin, kout, vout) == 0
    print(json.dumps(line), flush=True)


def run_fs(args, rank, world, local_rank):
    import numpy as np
    import torch

    import datagen
    import paper_2605_10390_b200 as fs
    from paper_2605_10390_b200 import _lib

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if args.workload == "c5":
        return run_fs_pairs(args, dev)
    L = fs.lib()
    dist_name, n_default, workload_text = WORKLOADS[args.workload]
    n = args.n or n_default
    if args.workload == "c4":  # fixed total, split over the ranks
        n_total = n
        n = n_total // world
    n_total = n * world
    i0 = rank * n
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream

    keys = torch.empty(n, dtype=torch.uint16, device=dev)
    if dist_name == "sortedswap":
        keys.copy_(torch.from_numpy(datagen.gen_u16("sortedswap", n_total, seed=0)[i0:i0 + n]))
    else:
        datagen.gen_u16_device(keys.data_ptr(), dist_name, n, seed=0, i0=i0, n_total=n_total, stream=s)
    out = torch.empty(n, dtype=torch.uint16, device=dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        prefix2 = torch.empty(65536 + 128, dtype=torch.int64, device=dev)
        htemp = torch.empty(L.fs_histogram_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
        b0, b1 = (n_total * rank) // world, (n_total * (rank + 1)) // world
    else:
        temp = torch.empty(L.fs_sort_keys_u16_temp_bytes(n), dtype=torch.uint8, device=dev)
    nev = 4
    # Phase events on every PHASE_EVERY-th timed step (a sample of the timed
    # region); the whole region is bracketed by t_begin / t_end.  Recording
    # events at every boundary of every step adds a few us per step.
    sampled = list(range(0, args.steps, PHASE_EVERY))
    events = {k: [torch.cuda.Event(enable_timing=True) for _ in range(nev)] for k in sampled}
    for row in events.values():
        for e in row:
            e.record(stream)  # materialise the cudaEvent_t handles
    handles = {k: ctypes_array(row) for k, row in events.items()}
    t_begin, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()

    def step(ev_row=None, ev_handles=None):
        if world == 1:
            if ev_handles is not None:
                L.fs_set_phase_events(ev_handles, nev)
            _lib.check(L.fs_sort_keys_u16(keys.data_ptr(), out.data_ptr(), n, 16, temp.data_ptr(), temp.numel(), s),
                       "fs_sort_keys_u16")
            if ev_handles is not None:
                L.fs_set_phase_events(None, 0)
        else:
            if ev_row is not None:
                ev_row[0].record(stream)
            _lib.check(L.fs_histogram_prefix_u16(keys.data_ptr(), n, prefix2.data_ptr(), htemp.data_ptr(),
                                                 htemp.numel(), s), "fs_histogram_prefix_u16")
            if ev_row is not None:
                ev_row[1].record(stream)
            # NCCL, 513 KiB: the global histogram merge across GPUs, in the
            # sort's two-level prefix form (linear in the counts: no scan after it)
            dist.all_reduce(prefix2)
            if ev_row is not None:
                ev_row[2].record(stream)
            _lib.check(L.fs_expand_prefix_u16(prefix2.data_ptr(), b0, b1, out.data_ptr(), s), "fs_expand_prefix_u16")
            if ev_row is not None:
                ev_row[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        t_begin.record(stream)
        for k in range(args.steps):
            step(events.get(k), handles.get(k))
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    total_ms = t_begin.elapsed_time(t_end)
    phase_ms = [statistics.mean(row[i].elapsed_time(row[i + 1]) for row in events.values()) for i in range(nev - 1)]
    t_max = total_ms
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    value = n_total * args.steps / (t_max * 1e-3) / 1e9

    # Roofline of the dominant kernel (algorithmic bytes = 2 B/key read for the
    # histogram, 2 B/key written for the expansion).
    if world == 1:
        names = {"hist16": phase_ms[1], "expand16": phase_ms[2]}  # phase 0 is empty (no memset)
        scan_ms = phase_ms[1]
    else:
        names = {"hist16+merge+scan": phase_ms[0], "expand16": phase_ms[2]}
        scan_ms = phase_ms[0]
    dom = max(names, key=names.get)
    dom_ms = names[dom]
    alg_bytes = 2 * (n if world == 1 else (b1 - b0) if dom == "expand16" else n)
    peak, peak_src = measured_peak_gbs()
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(dom.split("+")[0]) if (args.workload == "c2" and world == 1) else (None, None)
    whole_bytes = 4 * n
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": workload_text if (n == n_default or args.workload == "c4") else f"{n} uint16 keys per GPU, {dist_name}, seed 0",
                   "keys_per_gpu": n, "keys_total": n_total, "parallelism": f"dp{world}",
                   "multi_gpu_mode": None if world == 1 else "B (two-level prefix all-reduce + own-range expansion)",
                   "l2": (f"inputs ({n * 2 / 2**20:.0f} MiB/GPU) larger than L2 (126 MB): no flush between steps" if n * 2 > 126e6
                          else "L2-resident input (c1): launch-bound, no roofline claim")},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": round(dom_ms, 5),
                     "peak_source": peak_src, "traffic_source": traffic_src},
        "whole_step": {"algorithmic_bytes": whole_bytes, "achieved_GBps": round(whole_bytes / (t_max / args.steps * 1e-3) / 1e9, 1),
                       "frac_of_measured_peak": round(whole_bytes / (t_max / args.steps * 1e-3) / 1e9 / peak, 4),
                       "frac_of_8TBps": round(whole_bytes / (t_max / args.steps * 1e-3) / 8e12, 4)},
        "phases_ms": {k: round(v, 5) for k, v in zip(
            (["prologue", "hist16+merge+scan", "expand16"] if world == 1 else ["hist16+merge+scan", "nccl_allreduce", "expand16"]),
            phase_ms)},
        "gpu_launches": (1 if (world == 1 and n <= (1 << 18)) else 2) * args.steps,  # one cluster launch up to 2^18
        "clocks": clocks.summary(),
        "phase_events": f"recorded on every {PHASE_EVERY}th of the {args.steps} timed steps ({len(events)} steps); "
                        "ms_per_step from events bracketing the whole timed region",
    }
    del scan_ms

    # End to end through the public host-buffer API: H2D of the step's keys from
    # pinned memory, the sort, D2H of the sorted keys, every step.
    if not args.no_e2e and args.workload == "c2":
        line["e2e"] = e2e(args, L, _lib, keys, n, n_total, rank, world, dev, dist)

    if args.workload == "c4":
        line["scaling"] = "strong"
    if not args.no_verify and world == 1:
        line["verified"] = verify(out, keys) if n <= (1 << 28) else verify_sampled(out, keys)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        v, reps, dt, ok = time_oracle(n, 3, 0, min_seconds=10.0)
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
                                "sample": f"the full c2 input (2^28 keys) sorted {reps} times ({dt:.1f} s) by the "
                                          f"single-threaded C oracle", "cpu": cpu_model(), "host_cores": host_cores()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def ctypes_array(events):
    import ctypes
    arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
    return arr


def e2e(args, L, _lib, keys, n, n_total, rank, world, dev, dist):
    import torch
    steps = max(1, min(args.steps, 5))
    host_in = keys.cpu().pin_memory()
    host_out = torch.empty(n, dtype=torch.uint16).pin_memory()
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    if world == 1:
        work = torch.empty(L.fs_sort_keys_u16_host_work_bytes(n, 0), dtype=torch.uint8, device=dev)

        def one():
            _lib.check(L.fs_sort_keys_u16_host(host_in.data_ptr(), host_out.data_ptr(), n, 0, work.data_ptr(),
                                               work.numel(), s), "fs_sort_keys_u16_host")
        h2d, d2h = 2 * n, 2 * n
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
    one()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        one()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(n_total * steps / (ms * 1e-3) / 1e9, 4), "unit": "Gkeys/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "api": "fs_sort_keys_u16_host (pinned host buffers, batched copy/compute overlap)" if world == 1
            else "H2D + fs_histogram_prefix_u16 + NCCL all_reduce + fs_expand_prefix_u16 + D2H"}


def verify(out, keys):
    """Cheap end check of the timed output against the oracle (rank 0, N = 1)."""
    import numpy as np

    import oracle
    k = keys.cpu().numpy()
    o = out.cpu().numpy()
    return bool(np.array_equal(o, oracle.sort_u16(k)))


def verify_sampled(out, keys, chunk=1 << 28):
    """Full-size check without a host copy of the sort (c4): the oracle histogram
    of the input (streamed in chunks) fixes P; every value's first and last
    position, 2^20 random positions, and non-decreasing order (device, chunked)
    must agree with it -- together they pin the sorted multiset."""
    import numpy as np
    import torch

    import oracle
    n = keys.numel()
    C = np.zeros(65536, dtype=np.uint64)
    for a in range(0, n, chunk):
        C += oracle.histogram_u16(keys[a:a + chunk].cpu().numpy())
    P = oracle.exclusive_scan(C)
    nonempty = np.nonzero(C)[0]
    pos = np.concatenate([P[nonempty], P[nonempty + 1] - 1,
                          np.random.default_rng(0).integers(0, n, 1 << 20).astype(np.uint64)])
    want = (np.searchsorted(P, pos, side="right") - 1).astype(np.int64)
    idx = torch.from_numpy(pos.astype(np.int64)).to(out.device)
    got = out.view(torch.int16)[idx].to(torch.int64).cpu().numpy() & 0xFFFF
    ok = bool(np.array_equal(got, want))
    for a in range(0, n - 1, chunk):
        b = min(a + chunk + 1, n)
        seg = out[a:b].view(torch.int16).to(torch.int32) & 0xFFFF
        ok &= bool((seg[1:] >= seg[:-1]).all().item())
    return ok


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
