"""GPU verifier (csrc/verify.cuh, mst_gpu_verify) against the oracle's
restatement of the reference's verify_mst (verify.cpp:15-57): the same flags
and weight on correct, short, cyclic, duplicated, swapped and reordered
results; out-of-range ids raise IndexError (std::out_of_range). The C++
drop-in test compares verify_mst_gpu with the reference's own verify_mst,
details line included (tests/cpp/test_dropin.cpp)."""
import numpy as np
import pytest

from conftest import GOLDEN, load_npz

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2005_06913_b200 as P
    return P


def _variants(ids, m, rng):
    ids = np.asarray(ids, dtype=np.int64)
    yield "exact", ids
    if ids.size:
        yield "short", ids[:-1]
        yield "reversed", ids[::-1].copy()
        d = ids.copy()
        d[-1] = d[0]
        yield "duplicate", d
        s = ids.copy()
        outside = np.setdiff1d(np.arange(m), ids)
        if outside.size:
            s[ids.size // 2] = outside[rng.integers(0, outside.size)]
            yield "swapped", s
        yield "extra", np.concatenate([ids, ids[:1]])
    yield "empty", ids[:0]


def _check(P, O, n, src, dst, w, rng):
    g = P.Graph(n, src, dst, w)
    k = O.kruskal(n, src, dst, w)
    oracle = P.MstResult(k.ids.astype(np.int64), k.total_weight, 0, 0.0)
    for name, ids in _variants(k.ids, len(src), rng):
        res = P.MstResult(ids, int(np.asarray(w, dtype=np.uint64)[ids].sum()) if ids.size else 0, 0, 0.0)
        want = O.verify(n, src, dst, w, ids.astype(np.uint32))
        for orc in (oracle, None):
            rep = P.verify_mst(g, res, orc)
            assert rep.edge_count_ok == want["edge_count_ok"], name
            assert rep.is_acyclic == want["is_acyclic"], name
            assert rep.is_spanning == want["is_spanning"], name
            assert rep.weight == want["total_weight"], name
            if orc is None:
                assert rep.weight_matches_oracle is None and rep.edge_set_matches_oracle is None
            else:
                assert rep.weight_matches_oracle == (want["total_weight"] == k.total_weight), name
                same = sorted(ids.tolist()) == k.ids.tolist()
                assert rep.edge_set_matches_oracle == same, name
                want_ok = (want["edge_count_ok"] and want["is_acyclic"] and want["is_spanning"]
                           and rep.weight_matches_oracle and same)
                assert rep.all_ok() == want_ok, name


def test_verifier_matches_oracle_flags(P, oracle_mod):
    rng = np.random.default_rng(3)
    for name in ["gen_3000_6_2", "gen_1500_4_13", "multi_mid", "gen_100_3_5"]:
        z = load_npz(GOLDEN / f"{name}.npz")
        _check(P, oracle_mod, int(z["n"]), z["src"], z["dst"], z["w"], rng)
    # disconnected input, self-loops and parallel edges
    _check(P, oracle_mod, 7, np.array([0, 1, 0, 3, 4, 3, 5, 5], np.uint32),
           np.array([1, 2, 2, 4, 5, 5, 5, 3], np.uint32), np.array([1, 2, 3, 4, 5, 6, 0, 1], np.uint32), rng)


def test_verifier_out_of_range(P):
    g = P.Graph(3, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([1, 2], np.uint32))
    with pytest.raises(IndexError):
        P.verify_mst(g, P.MstResult(np.array([0, 2]), 3, 0, 0.0))
    with pytest.raises(IndexError):
        P.verify_mst(g, P.MstResult(np.array([-1, 0]), 3, 0, 0.0))


def test_verifier_aos_64bit_weights(P, oracle_mod):
    # the AoS entry sums the reference's full u64 weights
    rng = np.random.default_rng(5)
    n, m = 5000, 30000
    src = np.concatenate([np.arange(1, n), rng.integers(0, n, m - n + 1)]).astype(np.uint32)
    dst = np.concatenate([rng.integers(0, np.arange(1, n)), rng.integers(0, n, m - n + 1)]).astype(np.uint32)
    w32 = rng.permutation(m).astype(np.uint32)
    k = oracle_mod.kruskal(n, src, dst, w32)
    e = np.zeros(m, dtype=P.EDGE_DTYPE)
    e["src"], e["dest"] = src, dst
    e["weight"] = w32.astype(np.uint64) * (1 << 33) + 7  # order-preserving, > 2^32
    total = int(e["weight"][k.ids].sum(dtype=np.uint64))
    res = P.MstResult(k.ids.astype(np.int64), total, 0, 0.0)
    rep = P.verify_mst_aos(n, e, res, res)
    assert rep.all_ok() and rep.weight == total
    bad = P.MstResult(k.ids[:-1].astype(np.int64), total, 0, 0.0)
    rep = P.verify_mst_aos(n, e, bad, res)
    assert not rep.all_ok() and not rep.is_spanning and rep.components == 2


def test_verifier_full_size_c1(P):
    # the engine's own c1 result verifies clean against itself structurally
    from paper_2005_06913_b200 import configs as C
    g = C.generate_host(C.CONFIGS["c1"])
    r = P.boruvka_gpu(g)
    rep = P.verify_mst(g, r)
    assert rep.is_spanning and rep.is_acyclic and rep.edge_count_ok and rep.weight == r.total_weight
    assert rep.all_ok()
    rep = P.verify_mst(g, r, r)
    assert rep.all_ok()
