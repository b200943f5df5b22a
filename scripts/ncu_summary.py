"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
         --tag r01 --out profiles/

Writes profiles/ncu_summary_<tag>.md (key metrics and top stall reasons per
kernel, per-kernel share of the launch list) and profiles/ncu_traffic_<tag>.json
(dram__bytes_read.sum + dram__bytes_write.sum per launch, read by bench.py for
the roofline "traffic" field).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__waves_per_multiprocessor", "waves/SM"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "SMEM atomic wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "SMEM atomic bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    base = name.split("(")[0]
    return base.split("::")[-1].split("<")[0]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            v = v / 1000.0 if r[ui] in ("nsecond", "ns") else (v * 1000.0 if r[ui] in ("msecond", "ms") else v)  # -> us
            per[short(r[ki])].append(v)
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--note", default="")
    ap.add_argument("--alias", default="", help="name#i=alias,... renames the i-th launch of a kernel")
    a = ap.parse_args()
    h, units, rows = raw(a.rep)
    lines = [f"# ncu summary {a.tag}", "", a.note, "",
             f"Source: `{os.path.basename(a.rep)}` (ncu --set full --clock-control none; caches flushed per replay).", ""]
    traffic = {}
    alias = dict(x.split("=") for x in a.alias.split(",") if x)
    seen = defaultdict(int)
    for r in rows:
        k = short(r[h.index("Kernel Name")])
        kk = f"{k.replace('k_', '')}#{seen[k]}"
        seen[k] += 1
        k = alias.get(kk, k)
        lines.append(f"## {k}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| {label} (`{m}`) | {r[i]} | {units[i]} |")
                vals[m] = (r[i], units[i])
        rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * UNIT_SCALE.get(vals["dram__bytes_read.sum"][1], 1)
        wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * UNIT_SCALE.get(vals["dram__bytes_write.sum"][1], 1)
        traffic[k.replace("k_", "")] = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                                        "source": os.path.basename(a.rep)}
        stall = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued")]
        top = sorted(((float(r[h.index(c)] or 0), c) for c in stall), reverse=True)[:6]
        lines.append("")
        lines.append("Top warp-stall samples: " + ", ".join(
            f"{c.replace('smsp__pcsamp_warps_issue_stalled_', '')} {int(v)}" for v, c in top))
        lines.append("")
    if a.launches:
        per = launches(a.launches)
        tot = sum(sum(v) for v in per.values())
        lines += ["## Launch list (cold-cache, serialised; compare shares)", "", "| kernel | launches | mean us | share |",
                  "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot:.1%} |")
    os.makedirs(a.out, exist_ok=True)
    open(os.path.join(a.out, f"ncu_summary_{a.tag}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(a.out, f"ncu_traffic_{a.tag}.json"), "w"), indent=1)
    print("wrote", os.path.join(a.out, f"ncu_summary_{a.tag}.md"))


if __name__ == "__main__":
    main()
