"""Top SASS instructions of an ncu source page by stall samples / global traffic."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
print("total samples", tot)
key = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
for r in sorted(data, key=lambda r: -f(r, key))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{r[ix['Address']]:>6} {100*f(r,'Warp Stall Sampling (All Samples)')/tot:5.1f}% exec={f(r,'Instructions Executed'):>10.0f} "
          f"l1req={f(r,'L1 Tag Requests Global'):>9.0f} l2sec={f(r,'L2 Theoretical Sectors Global'):>10.0f} "
          f"lsb={f(r,'stall_long_sb'):>6.0f} membar={f(r,'stall_membar'):>6.0f} | {r[ix['Source']][:70]}")
