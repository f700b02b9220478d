"""Per-CUDA-source-line warp-stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass -k <kernel>`:
aggregates the SASS rows under each source line and prints the top lines
with their dominant stall reasons."""
import csv
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
ci = {}
for i, h in enumerate(hdr):
    ci.setdefault(h, i)
key = "Warp Stall Sampling (All Samples)"
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
agg = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0] not in ("", "-"):
        cur = int(r[0]) if r[0].isdigit() else cur
        src[cur] = r[1]
    if cur is None:
        continue
    agg[cur] += f(r[ci[key]])
    for i in stall_cols:
        reasons[cur][hdr[i][6:]] += f(r[i])
tot = sum(agg.values()) or 1.0
for line, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    top = sorted(reasons[line].items(), key=lambda x: -x[1])[:2]
    rs = ",".join(f"{k}:{100 * s / max(v, 1):.0f}%" for k, s in top if s)
    print(f"{100 * v / tot:5.1f}% L{line:<5} {rs:<28} {src.get(line, '')[:70]}")
