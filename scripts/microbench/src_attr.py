"""Attribute an ncu source-page metric to CUDA source lines (mixed cuda,sass view
of a report captured with --import-source on and a -lineinfo build).
Usage: src_attr.py report.ncu-rep kernel_regex launch_skip "metric[,metric2]" [top]"""
import collections, csv, io, subprocess, sys
rep, kre, skip, metrics = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4].split(",")
top = int(sys.argv[5]) if len(sys.argv) > 5 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = None, None
agg = collections.defaultdict(lambda: [0.0] * len(metrics)); text = {}
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; idx = [hdr.index(m) for m in metrics]; continue
    if hdr is None or len(r) < len(hdr) or not r[0]: continue  # SASS rows: the line rows hold the sums
    key = (fname, r[0]); text[key] = r[1].strip()
    for j, i in enumerate(idx):
        try: agg[key][j] += float(r[i] or 0)
        except ValueError: pass
tot = [sum(v[j] for v in agg.values()) or 1 for j in range(len(metrics))]
print("  ".join(f"{m}: {t:.4g}" for m, t in zip(metrics, tot)))
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("  ".join(f"{x / t * 100:5.1f}%" for x, t in zip(v, tot)) + f"  {key[0]}:{key[1]}: {text[key][:90]}")
