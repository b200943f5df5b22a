"""bench.py's JSON line on the GPU (the driver's contract): one
line with the required keys, a roofline block whose fraction is its achieved /
peak, an e2e block with the copied bytes, clocks and a verified output -- for
the headline workload (c2) and the pairs workload (c5), short runs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"]


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def check_common(d, steps, warmup):
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["unit"] == "Gkeys/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["data"] == "synthetic" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 2e-3
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)


def test_bench_line_c2():
    d = run_bench("--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    check_common(d, 5, 3)
    assert d["dtype"] == "u16" and d["config"]["keys_per_gpu"] == 1 << 28
    # value is keys per second over the timed steps
    assert abs(d["value"] - (1 << 28) / (d["ms_per_step"] * 1e-3) / 1e9) / d["value"] < 0.01
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 2 << 28 and e["d2h_bytes_per_step"] == 2 << 28 and e["value"] > 0
    assert d["verified"] is True


def test_bench_line_c5():
    d = run_bench("--workload", "c5", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e")
    check_common(d, 2, 3)
    assert d["config"]["pairs"] == 1 << 29
    assert d.get("verified_invariants") is True
