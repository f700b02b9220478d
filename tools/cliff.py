"""Plain-loop timing of one uniform graph under a few knobs (MST_* env)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C

    n_, m_ = int(float(sys.argv[1])), int(float(sys.argv[2]))
    n, m, s, d, w = C.generate_torch(C.uniform(n_, m_, seed=0))
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for knobs in ({}, {"MST_DEDUP": "0"}, {"MST_TAIL_EDGES": "1.2e7"}, {"MST_TAIL_EDGES": "1.2e7", "MST_DEDUP": "0"},
                  {"MST_TAIL": "0"}):
        os.environ.update({"MST_FILTER": "0", **knobs})
        P.api.tuning_from_env()
        info = P.GpuRunInfo()
        for _ in range(3):
            P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st, info=info)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        print(f"{knobs}: {e0.elapsed_time(e1) / 5:.3f} ms rounds={info.rounds} launches={info.kernel_launches}")
        print("   edges", info.live_edges)
        print("   comps", info.live_comps, flush=True)
        for k in knobs:
            os.environ.pop(k)


if __name__ == "__main__":
    main()
