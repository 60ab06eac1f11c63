"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0, "hit": 0.0})
for i, mets in per.items():
    a = agg[names[i]]
    a["n"] += 1
    a["ns"] += mets.get("gpu__time_duration.sum", 0)
    a["rd"] += mets.get("dram__bytes_read.sum", 0)
    a["wr"] += mets.get("dram__bytes_write.sum", 0)
    a["hit"] += mets.get("lts__t_sector_hit_rate.pct", 0)
tot = sum(a["ns"] for a in agg.values())
print(f"{'kernel':44s} {'n':>4s} {'mean_us':>9s} {'share':>6s} {'dram_MB/launch':>14s} {'L2hit%':>6s}")
out = {}
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
    mb = (a["rd"] + a["wr"]) / a["n"] / 1e6
    print(f"{k[:44]:44s} {a['n']:4d} {a['ns']/a['n']/1e3:9.1f} {100*a['ns']/tot:5.1f}% {mb:14.1f} {a['hit']/a['n']:6.1f}")
    out[k] = {"launches": a["n"], "mean_us": a["ns"] / a["n"] / 1e3, "share": a["ns"] / tot,
              "dram_bytes_per_launch": (a["rd"] + a["wr"]) / a["n"], "l2_hit_pct": a["hit"] / a["n"]}
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
