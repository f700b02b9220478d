"""Plain loop vs Filter-Boruvka across densities (sets filter_mode's m/n rule)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C

    specs = [C.uniform(1 << 20, 4 << 20, seed=0), C.uniform(1 << 20, 6 << 20, seed=0),
             C.uniform(1 << 20, 8 << 20, seed=0), C.uniform(1 << 20, 12 << 20, seed=0),
             C.uniform(1 << 22, 32 << 20, seed=0), C.rmat(20, 4, seed=2), C.rmat(20, 8, seed=2),
             C.rmat(20, 16, seed=2), C.rmat(22, 8, seed=2), C.CONFIGS["c2"], C.CONFIGS["c0"]]
    for spec in specs:
        n, m, s, d, w = C.generate_torch(spec)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        res = []
        for f in ("0", "1"):
            os.environ["MST_FILTER"] = f
            P.api.tuning_from_env()
            for _ in range(3):
                P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 10)
        print(f"{spec.name:28s} n={n:>9} m={m:>10} m/n={m / n:5.1f}  plain {res[0]:7.3f} ms  filter {res[1]:7.3f} ms",
              flush=True)
        del s, d, w, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
