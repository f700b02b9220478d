"""Seeded synthetic inputs (CPU generator; the GPU generator's byte-equality
with it is a -m gpu test)."""
import numpy as np
import pytest

from paper_2005_06913_b200 import configs as C


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2005_06913_b200.build import build_library
    build_library(verbose=False)


def _is_spanning_tree(n, a, b):
    parent = np.arange(n)

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for x, y in zip(a.tolist(), b.tolist()):
        rx, ry = find(x), find(y)
        if rx == ry:
            return False
        parent[rx] = ry
    return len(a) == n - 1


def test_uniform_structure_and_determinism():
    spec = C.uniform(5000, 20000, seed=9)
    g = C.generate_host(spec, threads=3)
    assert g.n == 5000 and g.edge_count() == 20000
    assert np.all(g.src < g.n) and np.all(g.dst < g.n)
    assert np.all(g.src != g.dst)
    assert np.array_equal(np.sort(g.w), np.arange(20000, dtype=np.uint32))  # permutation of 0..m-1
    assert _is_spanning_tree(g.n, g.src[: g.n - 1], g.dst[: g.n - 1])      # tree edges first
    g2 = C.generate_host(spec, threads=1)
    assert np.array_equal(g.src, g2.src) and np.array_equal(g.dst, g2.dst) and np.array_equal(g.w, g2.w)
    g3 = C.generate_host(C.uniform(5000, 20000, seed=10))
    assert not np.array_equal(g.w, g3.w)


def test_grid_structure():
    g = C.generate_host(C.grid(7, 11, seed=1))
    assert g.n == 77 and g.edge_count() == 7 * 10 + 6 * 11
    pairs = {(min(a, b), max(a, b)) for a, b in zip(g.src.tolist(), g.dst.tolist())}
    assert len(pairs) == g.edge_count()
    for a, b in pairs:
        ra, ca = divmod(a, 11)
        rb, cb = divmod(b, 11)
        assert abs(ra - rb) + abs(ca - cb) == 1
    assert np.array_equal(np.sort(g.w), np.arange(g.edge_count(), dtype=np.uint32))


def test_c1_edge_count_exact():
    assert C.edge_count(C.CONFIGS["c1"]) == 2 * 2048 * 2047 == 8_384_512
    assert C.edge_count(C.CONFIGS["c0"]) == 4_000_000
    assert C.edge_count(C.CONFIGS["c3"]) == 268_435_456


def test_rmat_structure_and_skew():
    spec = C.rmat(12, 8, seed=2)
    m = C.edge_count(spec)
    g = C.generate_host(spec, threads=4)
    n = 1 << 12
    assert g.n == n and g.edge_count() == m
    assert n - 1 < m <= n - 1 + 8 * n
    assert np.all(g.src != g.dst)                    # self-loops dropped
    assert _is_spanning_tree(n, g.src[: n - 1], g.dst[: n - 1])
    assert np.array_equal(np.sort(g.w), np.arange(m, dtype=np.uint32))
    deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=n)
    assert deg[0] > 20 * np.median(deg)              # a=0.57: vertex 0 is the hub
    pairs = np.minimum(g.src, g.dst).astype(np.uint64) << 32 | np.maximum(g.src, g.dst)
    assert np.unique(pairs).size < m                 # duplicate pairs are kept
    g1 = C.generate_host(spec, threads=1)
    assert np.array_equal(g.src, g1.src) and np.array_equal(g.w, g1.w)


@pytest.mark.parametrize("spec", [C.uniform(5000, 20000, seed=9), C.grid(33, 47, seed=1), C.rmat(13, 8, seed=4),
                                  C.uniform(2, 1, seed=0), C.grid(1, 2, seed=3)], ids=lambda s: s.name)
def test_oracle_generator_matches_product_bytes(spec, oracle_mod):
    """The restated generator (oracle/gen_oracle.c: the checkers' input, no
    product library) makes the product host generator's bytes exactly."""
    g = C.generate_host(spec, threads=2)
    assert oracle_mod.gen_count(spec) == g.edge_count()
    n, s, d, w = oracle_mod.generate(spec, threads=3)
    assert n == g.n
    assert np.array_equal(s, g.src) and np.array_equal(d, g.dst) and np.array_equal(w, g.w)


def test_golden_answers_pin_the_configs(oracle_mod):
    """tests/golden/answers.json (tests/golden/make_answers.py): the input
    hashes of the small configs still match the restated generator, and the
    recorded answers are spanning trees of the right size."""
    import hashlib
    import json
    from conftest import GOLDEN
    ans = json.loads((GOLDEN / "answers.json").read_text())
    assert set(ans) >= {"c0", "c1", "c2", "c3", "c4"}
    for key in ("c0", "c1"):
        a = ans[key]
        n, s, d, w = oracle_mod.generate(C.CONFIGS[key])
        assert (n, s.size) == (a["n"], a["m"])
        for name, arr in (("src", s), ("dst", d), ("w", w)):
            assert hashlib.sha256(arr.astype("<u4").tobytes()).hexdigest() == a[f"{name}_sha256"]
        k = oracle_mod.kruskal(n, s, d, w)
        assert hashlib.sha256(k.ids.astype("<u4").tobytes()).hexdigest() == a["ids_sha256"]
        assert k.total_weight == a["total_weight"]
    for a in ans.values():
        assert a["count"] == a["n"] - 1
