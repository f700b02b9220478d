"""Sum MST_TIMELINE stderr lines (last MST of a run) per kernel name.
Usage: python tools/timeline_sum.py file [file2]"""
import re
import sys
from collections import OrderedDict


def parse(path):
    runs, cur = [], []
    for line in open(path):
        m = re.match(r"timeline\s+([\d.]+) us\s+\+\s*([\d.]+)\s+(\S+)", line)
        if not m:
            continue
        t, d, name = float(m.group(1)), float(m.group(2)), m.group(3)
        if name == "(mark)" and cur:
            runs.append(cur)
            cur = []
        name = re.sub(r"^_ZN6mstgpu\d+", "", name)
        name = re.sub(r"E[A-Z].*$", "", name)[:40]
        cur.append((name, d))
    runs.append(cur)
    agg = OrderedDict()
    for name, d in runs[-1]:
        agg[name] = agg.get(name, 0.0) + d
    return agg, sum(d for _, d in runs[-1])


files = sys.argv[1:]
res = [parse(f) for f in files]
names = list(OrderedDict.fromkeys(n for a, _ in res for n in a))
for n in names:
    print(f"{n:42s} " + " ".join(f"{a.get(n, 0.0):10.1f}" for a, _ in res))
print(f"{'total':42s} " + " ".join(f"{t:10.1f}" for _, t in res))
