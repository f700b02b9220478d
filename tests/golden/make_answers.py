"""Golden MST answers of the five BASELINE.json configs (c0..c4).

    python tests/golden/make_answers.py [--configs c0,c1,c2,c3,c4] [--ref-check c0,c1]

For each config: the input is built by the restated generator
(oracle/gen_oracle.c — the same bytes as the product's host and device
generators, tests/test_generators.py), the MST by the pinned C oracle's
Kruskal (oracle/mst_oracle.c, restating kruskal_oracle,
/root/reference/proj/src/boruvka_seq.cpp:121-143), checked structurally by
the restated verify_mst (verify.cpp:15-57: n-1 edges, acyclic, spanning).
``--ref-check`` also runs the UNCHANGED reference kruskal_oracle
(oracle/_ref, through the SURVEY §8(c) adapter) on the same graph and
requires the same edge set (the adapter's total = ours + (n-1) when it
shifts weights by one) — it needs the reference's ~50 B/edge of host RAM.

Output: tests/golden/answers.json — per config n, m, the MST edge count,
the u64 total weight, SHA-256 of the ascending u32 ids (little endian) and
of the input arrays (so a generator change is caught before a GPU run).
TEST INFRASTRUCTURE ONLY (the GPU parity test compares against this file).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent / "answers.json"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


def main() -> int:
    from oracle import oracle as O
    from paper_2005_06913_b200 import configs as C  # spec table only (plain data)

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
    ap.add_argument("--ref-check", default="")
    a = ap.parse_args()
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    ref_check = set(filter(None, a.ref_check.split(",")))
    for key in filter(None, a.configs.split(",")):
        spec = C.CONFIGS[key]
        t0 = time.time()
        n, src, dst, w = O.generate(spec)
        t1 = time.time()
        k = O.kruskal(n, src, dst, w)
        t2 = time.time()
        v = O.verify(n, src, dst, w, k.ids)
        assert v["edge_count_ok"] and v["is_acyclic"] and v["is_spanning"], v
        assert v["total_weight"] == k.total_weight
        entry = {"workload": spec.name, "n": int(n), "m": int(src.size), "count": int(k.ids.size),
                 "total_weight": int(k.total_weight), "ids_sha256": sha(k.ids),
                 "src_sha256": sha(src), "dst_sha256": sha(dst), "w_sha256": sha(w),
                 "oracle": "oracle/mst_oracle.c oracle_kruskal (restates boruvka_seq.cpp:121-143)",
                 "gen_s": round(t1 - t0, 1), "kruskal_s": round(t2 - t1, 1)}
        if key in ref_check:
            if not O.ref_available():
                raise SystemExit("--ref-check needs oracle/_ref/libmstref.so")
            r = O.ref_solve(n, src, dst, w, O.ALGO_KRUSKAL)
            same = np.array_equal(r.ids, k.ids)
            shift = r.total_weight - k.total_weight
            assert same and shift in (0, n - 1), (same, shift)
            entry["reference_kruskal"] = {"same_edge_set": True, "total_weight": int(r.total_weight),
                                          "weight_shift": int(shift), "m_prime": int(r.m_prime),
                                          "elapsed_ms": round(r.elapsed_ms, 1)}
        prev = data.get(key, {})
        if "reference_kruskal" in prev and "reference_kruskal" not in entry and prev.get("ids_sha256") == entry["ids_sha256"]:
            entry["reference_kruskal"] = prev["reference_kruskal"]
        data[key] = entry
        print(key, json.dumps(entry), flush=True)
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
        del src, dst, w, k
    return 0


if __name__ == "__main__":
    sys.exit(main())
