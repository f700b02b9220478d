"""The CPU oracle pinned against the reference (CPU only, no GPU)."""
import numpy as np
import pytest

from conftest import golden_gen_files, load_npz, small_cases

# kruskal_oracle(generate_graph(n, d, seed)) computed by
# the unchanged reference (presets from bench.cpp:41-50).
APP_B = {
    (10_000, 3, 103): 54_539_809,
    (10_000, 6, 106): 59_021_951,
    (10_000, 9, 109): 59_952_592,
    (100_000, 3, 1003): 5_460_175_173,
    (100_000, 6, 1006): 5_911_779_114,
    (100_000, 9, 1009): 5_981_724_212,
}


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c[0])
def test_oracle_small_golden(oracle_mod, case):
    name, n, src, dst, w, ids, total = case
    k = oracle_mod.kruskal(n, src, dst, w)
    assert k.ids.tolist() == ids and k.total_weight == total
    s = oracle_mod.boruvka_seq(n, src, dst, w)
    assert s.ids.tolist() == ids and s.total_weight == total


@pytest.mark.parametrize("path", golden_gen_files(), ids=lambda p: p.stem)
def test_oracle_generated_golden(oracle_mod, path):
    g = load_npz(path)
    n = int(g["n"])
    k = oracle_mod.kruskal(n, g["src"], g["dst"], g["w"])
    assert np.array_equal(k.ids, g["ids"])
    assert k.total_weight == int(g["total"])
    s = oracle_mod.boruvka_seq(n, g["src"], g["dst"], g["w"])
    assert np.array_equal(s.ids, g["ids"])
    v = oracle_mod.verify(n, g["src"], g["dst"], g["w"], k.ids)
    assert v["edge_count_ok"] and v["is_acyclic"] and v["is_spanning"]
    assert v["total_weight"] == k.total_weight


def test_app_b_known_answers_from_fixtures(oracle_mod):
    for (n, d, seed), total in APP_B.items():
        p = __import__("conftest").GOLDEN / f"gen_{n}_{d}_{seed}.npz"
        if not p.exists():
            continue
        g = load_npz(p)
        assert oracle_mod.kruskal(n, g["src"], g["dst"], g["w"]).total_weight == total


def test_app_b_known_answers_via_reference(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    for (n, d, seed), total in APP_B.items():
        src, dst, w = oracle_mod.ref_generate_graph(n, d, seed)
        assert oracle_mod.kruskal(n, src, dst, w).total_weight == total
        assert oracle_mod.ref_solve(n, src, dst, w).total_weight == total


def test_oracle_matches_reference_on_random_multigraphs(oracle_mod):
    """Zero weights, duplicate pairs and self-loops through the §8(c) adapter."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        m = int(rng.integers(n - 1, 6 * n))
        tree_a = np.arange(1, n)
        tree_b = np.array([rng.integers(0, i) for i in range(1, n)], dtype=np.int64)
        ea = rng.integers(0, n, m - (n - 1))
        eb = rng.integers(0, n, m - (n - 1))  # self-loops and duplicates allowed
        src = np.concatenate([tree_a, ea]).astype(np.uint32)
        dst = np.concatenate([tree_b, eb]).astype(np.uint32)
        w = rng.permutation(m).astype(np.uint32)
        k = oracle_mod.kruskal(n, src, dst, w)
        r = oracle_mod.ref_solve(n, src, dst, w)
        assert np.array_equal(k.ids, r.ids) and k.total_weight == r.total_weight
        c = oracle_mod.ref_solve(n, src, dst, w, oracle_mod.ALGO_CAS, threads=3)
        assert np.array_equal(c.ids, r.ids)
        # the adapter built once, solved repeatedly (bench.py's CPU legs)
        rg = oracle_mod.RefGraph(n, src, dst, w)
        for algo, t in ((oracle_mod.ALGO_KRUSKAL, 1), (oracle_mod.ALGO_SEQ, 1), (oracle_mod.ALGO_CAS, 2),
                        (oracle_mod.ALGO_CAS, 4)):
            x = rg.solve(algo, threads=t)
            assert np.array_equal(x.ids, r.ids) and x.total_weight == r.total_weight and x.m_prime == r.m_prime
        rg.close()


def test_min_edges_table(oracle_mod):
    rng = np.random.default_rng(3)
    n, m = 200, 1500
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    w = rng.integers(0, 50, m).astype(np.uint32)  # ties: broken by id
    got = oracle_mod.min_edges(n, src, dst, w)
    want = np.full(n, np.iinfo(np.uint64).max, dtype=np.uint64)
    for e in range(m):
        if src[e] == dst[e]:
            continue
        key = (int(w[e]) << 32) | e
        for v in (src[e], dst[e]):
            want[v] = min(int(want[v]), key)
    assert np.array_equal(got, want)


def test_oracle_disconnected_forest(oracle_mod):
    # two triangles, no bridge: a spanning forest of 4 edges
    src = np.array([0, 1, 0, 3, 4, 3], dtype=np.uint32)
    dst = np.array([1, 2, 2, 4, 5, 5], dtype=np.uint32)
    w = np.array([1, 2, 3, 4, 5, 6], dtype=np.uint32)
    k = oracle_mod.kruskal(6, src, dst, w)
    assert k.ids.tolist() == [0, 1, 3, 4]
    v = oracle_mod.verify(6, src, dst, w, k.ids)
    assert not v["is_spanning"] and v["is_acyclic"]


def test_oracle_range_error(oracle_mod):
    with pytest.raises(ValueError):
        oracle_mod.kruskal(3, np.array([0, 5]), np.array([1, 2]), np.array([1, 2]))
