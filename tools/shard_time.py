"""Sharded protocol on one GPU: device time of the emulated-shard loop
(shards run back to back on one stream, the allreduce is a min kernel) next
to the single-device loop, and the oracle check of its edge set."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--shards", default="1,2,4,8")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    import numpy as np
    import paper_2005_06913_b200 as P
    P.api.tuning_from_env()  # MST_* knobs of the A/B scripts
    from paper_2005_06913_b200 import configs as C

    g = C.generate_host(C.CONFIGS[a.config])
    ref = P.boruvka_gpu(g)
    info = P.GpuRunInfo()
    for _ in range(a.reps):
        P.boruvka_gpu(g, info=info)
    print(f"{a.config}: single-device loop {info.ms_device:.3f} ms device, rounds={info.rounds}")
    for s in [int(x) for x in a.shards.split(",")]:
        best = None
        for _ in range(a.reps):
            info = P.GpuRunInfo()
            e = P.boruvka_gpu_emulated(g, s, info=info)
            best = info.ms_device if best is None else min(best, info.ms_device)
        same = np.array_equal(e.mst_edges, ref.mst_edges) and e.total_weight == ref.total_weight
        print(f"  {s} emulated shard(s): {best:.3f} ms device, rounds={info.rounds}, "
              f"launches={info.kernel_launches}, identical={same}")


if __name__ == "__main__":
    main()
