"""Per-kernel summary of an ncu --set full report (raw page): duration,
DRAM bytes, achieved DRAM GB/s, L2/L1 throughput, occupancy, registers.
Usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def num(row, name, scale=1.0):
    try:
        v = float(row[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return None
    u = units[col[name]]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6,
            "ms": 1e-3, "s": 1.0, "usecond": 1e-6,
            "msecond": 1e-3, "second": 1.0}.get(u, 1.0)
    return v * mult * scale


out = []
for row in rows[2:]:
    name = row[col["Kernel Name"]].split("(")[0].replace("void ", "")
    dur = num(row, "gpu__time_duration.sum")
    rd = num(row, "dram__bytes_read.sum") or 0.0
    wr = num(row, "dram__bytes_write.sum") or 0.0
    out.append({
        "kernel": name, "duration_us": dur * 1e6 if dur else None, "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_gbs": (rd + wr) / dur / 1e9 if dur else None,
        "dram_pct": num(row, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_pct": num(row, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l1_pct": num(row, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "occupancy_pct": num(row, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num(row, "launch__registers_per_thread"),
    })
tot_t = sum(o["duration_us"] or 0 for o in out)
print(f"{len(out)} kernels, {tot_t:.1f} us (ncu, serialised, cold L2 per replay)")
print(f"{'kernel':46s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>7s} {'dram%':>6s} {'L2%':>6s} {'L1%':>6s} {'occ%':>6s} {'regs':>5s}")
for o in out:
    f = lambda v, fmt: (fmt % v) if v is not None else "-"
    print(f"{o['kernel'][:46]:46s} {f(o['duration_us'], '%8.1f')} {(o['dram_read_bytes'] + o['dram_write_bytes']) / 1e6:9.1f} "
          f"{f(o['dram_gbs'], '%7.0f')} {f(o['dram_pct'], '%6.1f')} {f(o['l2_pct'], '%6.1f')} {f(o['l1_pct'], '%6.1f')} "
          f"{f(o['occupancy_pct'], '%6.1f')} {f(o['registers'], '%5.0f')}")
if "--json" in sys.argv:
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
