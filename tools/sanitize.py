"""Small MSTs through every single-GPU mode, for compute-sanitizer memcheck."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C
    from oracle import oracle as O

    modes = [{}, {"MST_FILTER": "0"}, {"MST_FILTER": "1"}, {"MST_TAIL": "0"},
             {"MST_FILTER": "0", "MST_TAIL_EDGES": "1e9", "MST_TAIL_DEDUP": "1", "MST_TAIL_DEDUP_MIN": "0",
              "MST_TAIL_DEDUP_RATIO": "1"},
             {"MST_FILTER": "0", "MST_TAIL_EDGES": "2e4", "MST_LAZY_ROUND1": "1"},
             {"MST_FILTER": "0", "MST_TAIL_EDGES": "2e4", "MST_LAZY_ROUND1": "0"}]
    specs = [C.grid(200, 300, seed=1), C.uniform(50_000, 200_000, seed=3), C.uniform(60_000, 100_000, seed=4),
             C.rmat(14, 8, seed=2)]
    for spec in specs:
        g = C.generate_host(spec)
        k = O.kruskal(g.n, g.src, g.dst, g.w)
        for mode in modes:
            os.environ.update(mode)
            P.api.tuning_from_env()
            r = P.boruvka_gpu(g)
            for key in mode:
                os.environ.pop(key)
            ok = np.array_equal(r.mst_edges, k.ids.astype(np.int64)) and r.total_weight == k.total_weight
            print(f"{spec.name} {mode}: {'ok' if ok else 'MISMATCH'}", flush=True)
            assert ok
        e = P.boruvka_gpu_emulated(g, 3)
        assert np.array_equal(e.mst_edges, k.ids.astype(np.int64))


if __name__ == "__main__":
    main()
