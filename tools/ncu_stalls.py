"""Per-kernel summary of an ncu --set full raw CSV export (ncu -i rep --page raw
--csv): duration, DRAM bytes and GB/s, L2 hit rate, achieved occupancy,
registers, and the top warp-stall reasons (PC sampling).
Usage: python tools/ncu_stalls.py raw.csv [more.csv ...]"""
import csv
import sys


def num(r, col, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return None


for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    units = rows[1]
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("mstgpu::", "")
        dur = num(r, col, "gpu__time_duration.sum")
        du = units[col["gpu__time_duration.sum"]]
        dur_us = dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(du, 1.0)
        rd = num(r, col, "dram__bytes_read.sum") or 0
        wr = num(r, col, "dram__bytes_write.sum") or 0
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= mult.get(units[col["dram__bytes_read.sum"]], 1)
        wr *= mult.get(units[col["dram__bytes_write.sum"]], 1)
        ss = {}
        for h in hdr:
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                v = num(r, col, h)
                if v:
                    ss[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        tot = sum(ss.values()) or 1
        top = sorted(ss.items(), key=lambda x: -x[1])[:5]
        print(f"{name[:48]:48s} {dur_us:9.1f} us  DRAM {rd / 1e9:6.2f}+{wr / 1e9:5.2f} GB "
              f"({(rd + wr) / (dur_us * 1e-6) / 1e9:5.0f} GB/s)  L2 hit {num(r, col, 'lts__t_sector_hit_rate.pct') or 0:5.1f}%  "
              f"occ {num(r, col, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0:5.1f}%  "
              f"regs {num(r, col, 'launch__registers_per_thread') or 0:.0f}")
        print("    stalls: " + "  ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
