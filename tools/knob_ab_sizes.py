"""A/B of one knob setting against the defaults across graph sizes and
families (filter-mode graphs of 8 M - 270 M edges), device-resident ms/MST.
Usage: python tools/knob_ab_sizes.py MST_TAIL_START_C_D=0 [MORE=..]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C

    env = dict(kv.split("=") for kv in sys.argv[1:])
    specs = [C.uniform(1 << 20, 8 << 20, seed=0), C.uniform(1 << 20, 16 << 20, seed=0),
             C.uniform(1 << 22, 32 << 20, seed=0), C.uniform(1 << 23, 128 << 20, seed=0),
             C.rmat(18, 16, seed=2), C.rmat(20, 8, seed=2), C.rmat(20, 16, seed=2), C.rmat(22, 8, seed=2),
             C.rmat(24, 16, seed=2), C.CONFIGS["c2"], C.CONFIGS["c3"]]
    for spec in specs:
        n, m, s, d, w = C.generate_torch(spec)
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        res = []
        for e in ({}, env):
            P.api.tuning_from_env(e)
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
        print(f"{spec.name:28s} n={n:>9} m={m:>10}  default {res[0]:7.3f} ms  {' '.join(sys.argv[1:])} {res[1]:7.3f} ms "
              f"({(res[1] / res[0] - 1) * 100:+.1f} %)", flush=True)
        del s, d, w, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
