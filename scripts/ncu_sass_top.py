"""Top SASS instructions of one kernel in an ncu report by stall samples
(needs -lineinfo / --import-source).  python scripts/ncu_sass_top.py REP [kernel-substr] [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fn, hdr, recs = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] in ("Function Name", "Kernel Name"):
        fn = r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and fn and want in fn and len(r) == len(hdr):
        recs.append(dict(zip(hdr, r)))
if not recs:
    sys.exit("no rows")
key = "Warp Stall Sampling (All Samples)"
# one row per SASS address (a report with several launches repeats them)
merged = {}
for x in recs:
    a = x["Address"][-5:]
    if a in merged:
        merged[a][key] = str(float(merged[a][key] or 0) + float(x[key] or 0))
    else:
        merged[a] = dict(x)
recs = list(merged.values())
tot = sum(float(x[key] or 0) for x in recs)
print(f"{len(recs)} SASS rows, {tot:.0f} samples")
for x in sorted(recs, key=lambda x: -float(x[key] or 0))[:top]:
    print(f"{float(x[key]) / tot * 100:5.1f}%  {x['Address'][-5:]}  {x['Source'][:70]:70s} "
          f"exec={x.get('Instructions Executed', '')}")
