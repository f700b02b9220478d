"""Per-launch table of an ncu --csv launch list taken with tools/gpu/r2_prof2.sh's
metric set: duration, DRAM read/write, L2 sector hit rate, L2 read / red /
atom sectors, L1 global-load requests and wavefronts, warps active,
registers. Usage: python tools/launch_table2.py launches.csv [--json out.json]"""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[1:]:
    try:
        d.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass


def short(name):
    name = name.replace("unnamed>::", "").replace("void ", "")
    head = name.split("(")[0]
    return head[:40]


out = []
tot = 0.0
print(f"{'id':>4} {'kernel':40s} {'us':>8s} {'DRAM_R MB':>9s} {'DRAM_W MB':>9s} {'GB/s':>6s} {'L2hit%':>6s} "
      f"{'L2rd Msec':>9s} {'red Msec':>8s} {'atom Msec':>9s} {'ldreq M':>8s} {'wf M':>7s} {'wf/SMcyc':>8s} {'occ%':>5s} {'reg':>4s}")
for k, v in d.items():
    if v["k"].startswith(("unnamed>::k_gen", "unnamed>::k_rmat", "k_gen")):
        continue  # the input generator
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rd, wr = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
    wf = v.get("l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum", 0)
    cyc = t * 1e-6 * 1.965e9 * 148
    rec = {"id": int(k), "kernel": short(v["k"]), "us": t, "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
           "dram_GBs": (rd + wr) / (t * 1e-6) / 1e9 if t else 0, "l2_hit_pct": v.get("lts__t_sector_hit_rate.pct", 0),
           "l2_read_Msectors": v.get("lts__t_sectors_op_read.sum", 0) / 1e6,
           "l2_red_Msectors": v.get("lts__t_sectors_op_red.sum", 0) / 1e6,
           "l2_atom_Msectors": v.get("lts__t_sectors_op_atom.sum", 0) / 1e6,
           "l1_ld_requests_M": v.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 0) / 1e6,
           "l1_wavefronts_M": wf / 1e6, "wavefronts_per_sm_cycle": wf / cyc if cyc else 0,
           "warps_active_pct": v.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
           "registers": v.get("launch__registers_per_thread", 0),
           # sectors the L1 fetched from L2 (its miss path: ~1 per SM-cycle at most, tools/gather_bench.cu)
           "l1_miss_Msectors": v.get("l1tex__m_xbar2l1tex_read_sectors.sum", 0) / 1e6,
           "l1_miss_sectors_per_sm_cycle": v.get("l1tex__m_xbar2l1tex_read_sectors.sum", 0) / cyc if cyc else 0}
    out.append(rec)
    print(f"{k:>4} {rec['kernel']:40s} {t:8.1f} {rd / 1e6:9.1f} {wr / 1e6:9.1f} {rec['dram_GBs']:6.0f} "
          f"{rec['l2_hit_pct']:6.1f} {rec['l2_read_Msectors']:9.1f} {rec['l2_red_Msectors']:8.1f} "
          f"{rec['l2_atom_Msectors']:9.1f} {rec['l1_ld_requests_M']:8.1f} {wf / 1e6:7.1f} "
          f"{rec['wavefronts_per_sm_cycle']:8.2f} {rec['warps_active_pct']:5.1f} {rec['registers']:4.0f} "
          f"{rec['l1_miss_Msectors']:11.1f} {rec['l1_miss_sectors_per_sm_cycle']:9.2f}")
print(f"total (generator excluded): {tot / 1e3:.3f} ms (ncu, serialised, cold L2 per launch)")
if "--json" in sys.argv:
    json.dump({"source": sys.argv[1], "launches": out, "total_ms": tot / 1e3},
              open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
