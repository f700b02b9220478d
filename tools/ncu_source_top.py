"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv`
output (one kernel), with the dominant stall reason of each line."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
key = "Warp Stall Sampling (All Samples)"
tot = sum(f(r[ci[key]]) for r in data) or 1.0
stalls = [h for h in hdr if h.startswith("stall_")]
for r in sorted(data, key=lambda r: -f(r[ci[key]]))[:n]:
    top = max(stalls, key=lambda s: f(r[ci[s]])) if stalls else ""
    print(f"{f(r[ci[key]]) / tot * 100:5.1f}% {r[ci['Address']]:>6} {top[6:]:<16} {r[ci['Source']][:80]}")
