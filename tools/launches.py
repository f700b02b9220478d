"""Summarise an ncu --csv launch list: per-launch device time of the LAST MST
(the helper runs warm-up + measured MSTs; kernels of one MST end with
k_bitmap_emit)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        nm = d['Kernel Name'].split('(')[0].replace('void ', '').replace('mstgpu::', '').replace('<unnamed>::', '')
        out.append((nm[:60], float(d['Metric Value'])))
ends = [i for i, (k, _) in enumerate(out) if k.startswith(("k_bitmap_emit", "k_flags_emit"))]
start = ends[-2] + 1 if len(ends) >= 2 else 0
last = out[start:ends[-1] + 1]
tot = sum(v for _, v in last)
print(f"{len(last)} launches, {tot/1000:.1f} us total (ncu, serialised)")
agg = {}
for k, v in last:
    name = k.split('<')[0]
    agg[name] = agg.get(name, 0) + v
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {v/1000:9.1f} us {100*v/tot:5.1f}%  {k}")
if '-v' in sys.argv:
    for k, v in last:
        print(f"{v/1000:10.1f}  {k}")
