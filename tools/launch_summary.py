"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of `bench.py --quick`:
k_linear launches in stack order (qkv, o, gu, d per block) -> per-class mean/median and share.
usage: python tools/launch_summary.py launches.csv out.json "<command that produced it>" """
import csv
import json
import statistics
import sys

src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = []
with open(src) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if "k_linear" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum":
        rows.append((float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0), r["Block Size"], r["Grid Size"]))
classes = ["qkv", "o", "gu", "d"]
per = {c: [] for c in classes}
meta = {}
for i, (us, blk, grid) in enumerate(rows):
    c = classes[i % 4]
    per[c].append(us)
    meta[c] = (blk, grid)
total = sum(u for u, _, _ in rows)
res = {"source": cmd, "launches": len(rows),
       "note": "ncu serialises launches (no PDL overlap) and runs them cold: absolute times exceed the in-graph ones; the shares carry over",
       "per_class": {c: {"launches": len(v), "mean_us": round(statistics.mean(v), 2), "median_us": round(statistics.median(v), 2),
                         "share_of_step": round(sum(v) / total, 4), "block": meta[c][0], "grid": meta[c][1]}
                     for c, v in per.items() if v}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res["per_class"]))
