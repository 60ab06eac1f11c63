"""profiles/ncu_traffic.json from an ncu launch list of bench.py (the DRAM
bytes bench.py reports as roofline.traffic for its gather kernels):
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
        --clock-control none -k regex:'k_pull_hot|k_push_hub|k_hub_fold|k_pr_update2'
        -s 30 -c 8 --csv --log-file L.csv python bench.py --steps 2 --warmup 3 ...
    python scripts/ncu_traffic.py L.csv
"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[h]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = defaultdict(dict)
for r in rows[h + 1:]:
    per[(r[ii], r[ki].split("(")[0].replace("void ", "").strip())][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    key = next(k for k in ("k_pull_hot", "k_push_hub", "k_hub_fold", "k_pr_update2") if k in name)
    a = agg[key]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[2] += m.get("gpu__time_duration.sum", 0)
avg = {k: (v[1] / v[0], v[2] / v[0]) for k, v in agg.items()}
gather = sum(avg[k][0] for k in ("k_pull_hot", "k_push_hub", "k_hub_fold") if k in avg)
out = {
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "--clock-control none (scripts/ncu_traffic.py), bench.py rmat:24:16:1 W=2^23, "
              "degree-ordered + hybrid (20480 hubs); per launch: "
              + ", ".join(f"{k} {b / 1e9:.3f} GB / {t / 1e3:.0f} us" for k, (b, t) in sorted(avg.items())),
    "k_pull_hot_bytes_per_iteration": int(gather),
    "k_pull_hot_launches_per_iteration": 3,
    "k_pr_update2_bytes_per_launch": int(avg.get("k_pr_update2", (0, 0))[0]),
    "graph": "rmat:24:16:1",
    "width": 8388608,
    "note": "gather category = k_pull_hot (pull, A+C edges) + k_push_hub + k_hub_fold (hybrid "
            "hub-destination edges), one launch each per iteration",
}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
