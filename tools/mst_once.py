"""Profiling helper: generate a config on the GPU, run W warm-up MSTs and R
measured MSTs through the device-resident entry (for ncu / launch lists)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--reps", type=int, default=1)
    a = p.parse_args()
    import torch
    import paper_2005_06913_b200 as P
    P.api.tuning_from_env()  # MST_* knobs of the A/B scripts
    from paper_2005_06913_b200 import configs as C

    n, m, s, d, w = C.generate_torch(C.CONFIGS[a.config])
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    info = P.GpuRunInfo()
    for i in range(a.warmup + a.reps):
        if i == a.warmup:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st, info=info)
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.config}: {e0.elapsed_time(e1) / a.reps:.3f} ms/MST rounds={info.rounds} "
          f"launches/MST={info.kernel_launches}")
    print("  live_edges", info.live_edges)
    print("  live_comps", info.live_comps)


if __name__ == "__main__":
    main()
