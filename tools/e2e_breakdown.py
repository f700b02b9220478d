"""Where the end-to-end time of one MST through the public API goes (pinned
host arrays, as bench.py's e2e leg): host wall, H2D, device, D2H; plus raw
pinned copy rates (one stream vs one stream per array) for comparison."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--flush", action="store_true", help="512 MiB device write + sync before each call")
    a = p.parse_args()
    import numpy as np
    import torch
    import paper_2005_06913_b200 as P
    P.api.tuning_from_env()  # MST_* knobs of the A/B scripts
    from paper_2005_06913_b200 import configs as C

    g0 = C.generate_host(C.CONFIGS[a.config])
    m = g0.edge_count()
    pins = [torch.empty(m, dtype=torch.int32, pin_memory=True) for _ in range(3)]
    for t, arr in zip(pins, (g0.src, g0.dst, g0.w)):
        t.numpy().view(np.uint32)[:] = arr
    g = P.Graph(g0.n, *(t.numpy().view(np.uint32) for t in pins))
    info = P.GpuRunInfo()
    for _ in range(2):
        P.boruvka_gpu(g)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(a.reps):
        if a.flush:
            flush.zero_()
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.boruvka_gpu(g, info=info)
        wall = (time.perf_counter() - t0) * 1e3
        print(f"{a.config}: wall {wall:.3f} ms | lib total {info.ms_total:.3f} h2d {info.ms_h2d:.3f} "
              f"device {info.ms_device:.3f} d2h {info.ms_d2h:.3f}")
    dev = [torch.empty(m, dtype=torch.int32, device="cuda") for _ in range(3)]
    for mode in ("one stream", "three streams"):
        streams = [torch.cuda.Stream() for _ in range(3)]
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(3):
                s = streams[i] if mode == "three streams" else streams[0]
                with torch.cuda.stream(s):
                    dev[i].copy_(pins[i], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"  H2D {12 * m / 1e6:.1f} MB pinned, {mode}: {best * 1e3:.3f} ms = {12 * m / best / 1e9:.1f} GB/s")
    out = torch.empty(g0.n, dtype=torch.int32, pin_memory=True)
    src = torch.empty(g0.n, dtype=torch.int32, device="cuda")
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"  D2H {4 * g0.n / 1e6:.1f} MB pinned: {best * 1e3:.3f} ms = {4 * g0.n / best / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
