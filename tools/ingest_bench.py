"""Ingestion rates: binary SoA file -> HBM through
load_graph_device, and the reference text format through the parallel
parser, for one BASELINE config. Files go to --dir (default /tmp); the page
cache is warm after the write, so this measures the pinned-staging path, not
the disk."""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--dir", default="/tmp")
    p.add_argument("--text", action="store_true", help="also time the text format")
    a = p.parse_args()
    import torch
    import paper_2005_06913_b200 as P
    P.api.tuning_from_env()  # MST_* knobs of the A/B scripts
    from paper_2005_06913_b200 import configs as C

    g = C.generate_host(C.CONFIGS[a.config])
    m = g.edge_count()
    path = Path(a.dir) / f"ingest_{a.config}.mstb"
    t0 = time.perf_counter()
    P.save_graph(g, path, binary=True)
    t_save = time.perf_counter() - t0
    P.load_graph_device(path)  # warm-up (allocations, page cache)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        P.load_graph_device(path)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    gb = 12 * m / 1e9
    print(f"{a.config}: m={m} binary save {gb / t_save:.2f} GB/s, file->HBM {gb / best:.2f} GB/s "
          f"({best * 1e3:.1f} ms for {gb:.2f} GB)")
    os.unlink(path)
    if a.text:
        tp = Path(a.dir) / f"ingest_{a.config}.txt"
        t0 = time.perf_counter()
        P.save_graph(g, tp)
        t_ws = time.perf_counter() - t0
        size = tp.stat().st_size / 1e9
        t0 = time.perf_counter()
        h = P.load_graph(tp)
        t_rd = time.perf_counter() - t0
        assert h.edge_count() == m
        print(f"  text: {size:.2f} GB, write {size / t_ws:.2f} GB/s, parse {size / t_rd:.2f} GB/s "
              f"({m / t_rd / 1e6:.1f} M edges/s, {os.cpu_count()} host threads)")
        os.unlink(tp)


if __name__ == "__main__":
    main()
