"""A/B of one knob setting against the defaults across graph sizes and
families (filter-mode graphs of 8 M - 270 M edges, or with --plain the
plain-loop family: grids, sparse uniform / R-MAT), device-resident ms/MST.
Usage: python tools/knob_ab_sizes.py [--plain] MST_TAIL_START_C_D=0 [MORE=..]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C

    plain = "--plain" in sys.argv  # the plain-loop family (m < 5 n): grids, sparse uniform / R-MAT graphs
    sys.argv = [a for a in sys.argv if a != "--plain"]
    env = dict(kv.split("=") for kv in sys.argv[1:])
    specs = [C.CONFIGS["c0"], C.CONFIGS["c1"], C.grid(1024, 1024, seed=1), C.grid(4096, 4096, seed=1),
             C.grid(512, 16384, seed=1), C.uniform(1 << 22, 3 << 22, seed=0), C.uniform(1 << 24, 1 << 26, seed=0),
             C.rmat(20, 2, seed=2), C.rmat(22, 3, seed=2), C.rmat(24, 2, seed=2)] if plain else [C.uniform(1 << 20, 8 << 20, seed=0), C.uniform(1 << 20, 16 << 20, seed=0),
             C.uniform(1 << 22, 32 << 20, seed=0), C.uniform(1 << 23, 128 << 20, seed=0),
             C.rmat(18, 16, seed=2), C.rmat(20, 8, seed=2), C.rmat(20, 16, seed=2), C.rmat(22, 8, seed=2),
             C.rmat(24, 16, seed=2), C.CONFIGS["c2"], C.CONFIGS["c3"]]
    def lattice(name, dims, offsets):
        """Lattice built with torch on the device: vertices of a dims box, an
        edge along each offset vector (3-D grid, 8-neighbour 2-D grid, ...),
        weights a random permutation."""
        idx = torch.arange(int(torch.tensor(dims).prod()), device="cuda", dtype=torch.int64)
        coords, rem = [], idx
        for dsz in reversed(dims):
            coords.append(rem % dsz)
            rem = rem // dsz
        coords = coords[::-1]
        srcs, dsts = [], []
        for off in offsets:
            ok = torch.ones_like(idx, dtype=torch.bool)
            tgt = torch.zeros_like(idx)
            for c, o, dsz in zip(coords, off, dims):
                ok &= (c + o >= 0) & (c + o < dsz)
                tgt = tgt * dsz + (c + o)
            srcs.append(idx[ok])
            dsts.append(tgt[ok])
        s_, d_ = torch.cat(srcs).to(torch.int32), torch.cat(dsts).to(torch.int32)
        w_ = torch.randperm(s_.numel(), device="cuda").to(torch.int32)
        return name, idx.numel(), s_.numel(), s_, d_, w_

    class _Named:
        def __init__(self, name):
            self.name = name

    if plain:
        specs += [lambda: lattice("grid3d_256^3", (256, 256, 256), [(1, 0, 0), (0, 1, 0), (0, 0, 1)]),
                  lambda: lattice("grid2d_8nbr_4096^2", (4096, 4096), [(1, 0), (0, 1), (1, 1), (1, -1)]),
                  lambda: lattice("grid2d_8nbr_2048^2", (2048, 2048), [(1, 0), (0, 1), (1, 1), (1, -1)]),
                  lambda: lattice("grid3d_128^3", (128, 128, 128), [(1, 0, 0), (0, 1, 0), (0, 0, 1)])]
    for spec in specs:
        if callable(spec):
            name, n, m, s, d, w = spec()
            spec = _Named(name)
        else:
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
