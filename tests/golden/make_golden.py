"""Generate the golden fixtures under tests/golden/ from the UNCHANGED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Every expected answer comes from the reference library compiled by
oracle/Makefile (oracle/_ref/libmstref.so): its generate_graph for the
graphs, its kruskal_oracle (through the SURVEY §8(c) adapter) for the
answers, cross-checked against its boruvka_seq and boruvka_cas, and, for the
tiny graphs, against an exhaustive brute force (the reference test suite's
own oracle shape, proj/tests/brute_force.hpp:22-64).
"""
from __future__ import annotations

import itertools
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent


def solve_all(n, src, dst, w):
    k = O.ref_solve(n, src, dst, w, O.ALGO_KRUSKAL)
    s = O.ref_solve(n, src, dst, w, O.ALGO_SEQ)
    c = O.ref_solve(n, src, dst, w, O.ALGO_CAS, threads=4)
    assert np.array_equal(k.ids, s.ids) and np.array_equal(k.ids, c.ids), "reference paths disagree"
    assert k.total_weight == s.total_weight == c.total_weight
    return k


def brute_force(n, src, dst, w):
    """Exhaustive minimum over all (n-1)-subsets (brute_force.hpp:22-64)."""
    m = len(src)
    best = None
    for combo in itertools.combinations(range(m), n - 1):
        par = list(range(n))

        def root(v):
            while par[v] != v:
                v = par[v]
            return v

        ok = True
        for e in combo:
            a, b = root(int(src[e])), root(int(dst[e]))
            if a == b:
                ok = False
                break
            par[a] = b
        if not ok:
            continue
        tot = sum(int(w[e]) for e in combo)
        if best is None or tot < best[0]:
            best = (tot, list(combo))
    return best


def hand_graphs():
    # the reference tests' hand graphs (test_boruvka_seq.cpp:17-26,40-78,134-140)
    return {
        "triangle": (3, [(0, 1, 1), (1, 2, 2), (0, 2, 3)]),
        "path": (3, [(0, 1, 4), (1, 2, 9)]),
        "k4": (4, [(0, 1, 1), (0, 2, 2), (0, 3, 3), (1, 2, 4), (1, 3, 5), (2, 3, 6)]),
        "star": (5, [(0, 1, 1), (0, 2, 2), (0, 3, 3), (0, 4, 4)]),
        "single_edge": (2, [(0, 1, 7)]),
    }


def small_random(count=200, seed=7):
    """Random connected graphs, n in 2..7, <= 12 edges, distinct weights
    (the shape of test_boruvka_seq.cpp:80-117; our own RNG)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(2, 8))
        edges, pairs = [], set()
        for i in range(1, n):
            j = int(rng.integers(0, i))
            pairs.add((min(i, j), max(i, j)))
            edges.append([i, j])
        for _ in range(int(rng.integers(0, 5))):
            if len(edges) >= 12:
                break
            a, b = int(rng.integers(0, n)), int(rng.integers(0, n))
            if a == b or (min(a, b), max(a, b)) in pairs:
                continue
            pairs.add((min(a, b), max(a, b)))
            edges.append([a, b])
        perm = rng.permutation(len(edges)) + 1
        out.append((n, [(a, b, int(wt)) for (a, b), wt in zip(edges, perm)]))
    return out


def multigraph_cases():
    """BASELINE-style inputs the reference's build_graph rejects raw: zero
    weights, duplicate pairs, self-loops (solved through the adapter)."""
    rng = np.random.default_rng(11)
    cases = {}
    for name, n, m in [("multi_small", 50, 400), ("multi_mid", 2000, 12000)]:
        tree_a = np.arange(1, n)
        tree_b = np.array([rng.integers(0, i) for i in range(1, n)])
        extra_a = rng.integers(0, n, m - (n - 1))
        extra_b = rng.integers(0, n, m - (n - 1))
        src = np.concatenate([tree_a, extra_a]).astype(np.uint32)
        dst = np.concatenate([tree_b, extra_b]).astype(np.uint32)
        w = rng.permutation(m).astype(np.uint32)  # 0..m-1, distinct
        cases[name] = (n, src, dst, w)
    return cases


def main():
    assert O.ref_available(), "build oracle/_ref first: make -C oracle ref"
    small = {}
    for name, (n, edges) in hand_graphs().items():
        a = np.array(edges, dtype=np.uint64)
        r = solve_all(n, a[:, 0], a[:, 1], a[:, 2])
        small[name] = {"n": n, "edges": edges, "ids": r.ids.tolist(), "total": r.total_weight}
    rand = []
    for n, edges in small_random():
        a = np.array(edges, dtype=np.uint64)
        r = solve_all(n, a[:, 0], a[:, 1], a[:, 2])
        bf = brute_force(n, a[:, 0], a[:, 1], a[:, 2])
        assert bf[0] == r.total_weight and sorted(bf[1]) == r.ids.tolist()
        rand.append({"n": n, "edges": edges, "ids": r.ids.tolist(), "total": r.total_weight})
    small["random200"] = rand
    (OUT / "small_graphs.json").write_text(json.dumps(small, separators=(",", ":")))

    # generate_graph instances used by the reference's own tests
    # (test_boruvka_parallel.cpp:49-137, test_boruvka_seq.cpp:119-163) and
    # the Graph10K presets (bench.cpp:41-50).
    gens = [(3000, 6, 2), (3000, 6, 5), (10000, 6, 2), (2000, 5, 21), (1500, 4, 13), (800, 4, 99),
            (1000, 6, 11), (100, 3, 5), (200, 4, 3), (10000, 3, 103), (10000, 6, 106),
            (10000, 9, 109)]
    for n, d, seed in gens:
        src, dst, w = O.ref_generate_graph(n, d, seed)
        r = solve_all(n, src, dst, w)
        np.savez_compressed(OUT / f"gen_{n}_{d}_{seed}.npz", n=n, src=src, dst=dst, w=w, ids=r.ids,
                            total=np.uint64(r.total_weight))
    for name, (n, src, dst, w) in multigraph_cases().items():
        r = solve_all(n, src, dst, w)
        np.savez_compressed(OUT / f"{name}.npz", n=n, src=src, dst=dst, w=w, ids=r.ids,
                            total=np.uint64(r.total_weight), m_prime=np.uint64(r.m_prime))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
