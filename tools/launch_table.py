"""Per-launch table (duration, DRAM read/write) of an ncu --csv launch list
taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.
Usage: python tools/launch_table.py launches.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
tot = 0.0
for k, v in d.items():
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    if v["k"].startswith(("unnamed>::k_gen", "unnamed>::k_rmat", "k_gen")):
        continue  # the input generator
    tot += t
    print(f"{k:>3} {v['k'][:56]:56s} {t:9.1f} us  R {v.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB"
          f"  W {v.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
print(f"total (generator excluded): {tot / 1e3:.2f} ms (ncu, serialised)")
