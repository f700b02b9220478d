"""Where bench.py's e2e wall time goes outside the library call: times
_host_out (torch pinned allocation), the C call and result wrapping, with
and without the previous result kept alive."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import paper_2005_06913_b200 as P
    P.api.tuning_from_env()  # MST_* knobs of the A/B scripts
    from paper_2005_06913_b200 import api as A
    from paper_2005_06913_b200 import configs as C

    n, m, s, d, w = C.generate_torch(C.CONFIGS["c1"], device="cuda:0")
    hs, hd, hw = (torch.empty(m, dtype=torch.int32, pin_memory=True) for _ in range(3))
    hs.copy_(s), hd.copy_(d), hw.copy_(w)
    g = P.Graph(n, hs.numpy().view(np.uint32), hd.numpy().view(np.uint32), hw.numpy().view(np.uint32))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for keep in (True, False):
        r = None
        for i in range(8):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            buf = A._host_out(n - 1)
            t1 = time.perf_counter()
            del buf
            info = P.GpuRunInfo()
            t2 = time.perf_counter()
            rr = P.boruvka_gpu(g, info=info)
            t3 = time.perf_counter()
            if keep:
                r = rr
            del rr
            print(f"keep={keep} i={i}: host_out {1e3*(t1-t0):.3f} ms | call {1e3*(t3-t2):.3f} ms "
                  f"(lib {info.ms_total:.3f})", flush=True)


if __name__ == "__main__":
    main()
