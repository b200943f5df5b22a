"""bench.py's reference arm (the CPU oracle, this tier's reference) prints one
well-formed JSON line on a CPU-only box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Gkeys/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["verified_nondecreasing"] is True


def test_roofline_traffic_comes_from_the_workloads_own_capture():
    """The roofline's `traffic` (ncu DRAM bytes per launch) is read from the newest
    committed capture OF THE SAME WORKLOAD: c2's hist16 never takes c3a's numbers
    (different input, different kernel path), and a workload without a capture
    reports none."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    t, src = bench.load_traffic("hist16", "c2")
    assert src is not None and not src.endswith(("_c3a.json", "_c5.json")) and t > 0
    t, src = bench.load_traffic("hist16", "c3a")
    assert src is not None and src.endswith("_c3a.json")
    assert bench.load_traffic("hist16", "c1") == (None, None)
    t, src = bench.load_traffic("local_sort", "c5")
    assert src is not None and t > 0
