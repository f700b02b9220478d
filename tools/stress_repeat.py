"""Race / flakiness stress: R back-to-back MSTs of a BASELINE config through
the device-resident entry, every result checked against the oracle's golden
answer (tests/golden/answers.json: count, u64 total, SHA-256 of the ascending
ids). A timing-dependent bug (grid-sync ordering in the tail, look-back
epochs, workspace reuse) shows up as a mismatch in some repetition.
Usage: python tools/stress_repeat.py --config c1 --reps 200 [MST_* knobs in the environment]"""
import argparse
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--reps", type=int, default=100)
    a = p.parse_args()
    import torch
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C
    P.api.tuning_from_env()
    ans = json.loads((ROOT / "tests/golden/answers.json").read_text())[a.config]
    n, m, s, d, w = C.generate_torch(C.CONFIGS[a.config])
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    bad = 0
    for i in range(a.reps):
        out.zero_()
        count, total = P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(), st)
        ids = out[:count].cpu().numpy().view(np.uint32)
        sha = hashlib.sha256(np.ascontiguousarray(ids).astype("<u4", copy=False).tobytes()).hexdigest()
        ok = count == ans["count"] and total == ans["total_weight"] and sha == ans["ids_sha256"]
        if not ok:
            bad += 1
            print(f"{a.config} rep {i}: MISMATCH count={count} total={total}")
    print(f"{a.config}: {a.reps} MSTs, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
