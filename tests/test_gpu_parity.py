"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bit-exact: the MST edge-id set and the u64 total weight (integer work, no
tolerance). Run on a B200 with `pytest -m gpu`.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_gen_files, load_npz, small_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mst():
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import _lib as L
    assert L.lib().mst_gpu_device_count() > 0, "no CUDA device: -m gpu tests need a B200"
    return P


def _env(**kv):
    """Force engine knobs for the calls inside (the library's tuning table,
    include/mst_gpu.h; the library never reads the environment)."""
    from paper_2005_06913_b200 import api
    return api.tuning(**kv)


# plain round loop, and Filter-Boruvka with a small / default / large light set
MODES = [dict(MST_FILTER=0), dict(MST_FILTER=1, MST_FILTER_BETA=0.3),
         dict(MST_FILTER=1, MST_FILTER_BETA=2), dict(MST_FILTER=1, MST_FILTER_BETA=50),
         # every round through the separate kernels with the pair-dedup variant armed
         dict(MST_FILTER=0, MST_TAIL=0, MST_DEDUP_MIN_EDGES=0),
         dict(MST_FILTER=1, MST_TAIL=0, MST_DEDUP_MIN_EDGES=0),
         # the tail megakernel with one block per SM (other chunk sizes)
         dict(MST_FILTER=0, MST_TAIL_BPS=1, MST_TAIL_EDGES=1e9),
         # the tail without its one-sync tiny rounds (three phases every round)
         dict(MST_FILTER=0, MST_TAIL_EDGES=1e9, MST_TAIL_TINY=0),
         # the tail's tagged pair dedup (opt-in) forced on in every round
         dict(MST_FILTER=0, MST_TAIL_EDGES=1e9, MST_TAIL_DEDUP=1, MST_TAIL_DEDUP_MIN=0, MST_TAIL_DEDUP_RATIO=1),
         dict(MST_FILTER=1, MST_TAIL_EDGES=1e9, MST_TAIL_DEDUP=1, MST_TAIL_DEDUP_MIN=0, MST_TAIL_DEDUP_RATIO=1),
         # round 1 compacted by the round kernels, then the tail (no start at phase C)
         dict(MST_FILTER=0, MST_TAIL_START_C=0),
         # round 1 compacted (no lazy pairs list), every round kernel offering batched / as plain REDs
         dict(MST_FILTER=0, MST_LAZY_ROUND1=0, MST_TAIL=0),
         dict(MST_FILTER=1, MST_TAIL=0, MST_OFFER_MIN1=2, MST_OFFER_SPLIT=2, MST_OFFER_COUNT=2, MST_OFFER_HEAVY=2),
         dict(MST_FILTER=0, MST_TAIL=0, MST_OFFER_MIN1=0, MST_OFFER_COUNT=0),
         # offer filter reads through L2 only (the default reads through L1), light phase without retirement
         dict(MST_FILTER=1, MST_TAIL=0, MST_OFFER_CACHED=0, MST_RETIRE=0),
         # the split's / heavy filter's offers as range passes over tiny table slices
         dict(MST_FILTER=1, MST_TAIL=0, MST_RANGE_MB=0.01),
         dict(MST_FILTER=1, MST_RANGE_MB=0.05, MST_OFFER_SPLIT=2, MST_OFFER_HEAVY=2),
         # the MST bitmap output (default above 64 Mi edges)
         dict(MST_FILTER=1, MST_TAIL=0, MST_BYTES_MAX=0),
         dict(MST_FILTER=0, MST_BYTES_MAX=0),
         # giant bits in every relabel round (default: >= 16 M components only)
         dict(MST_FILTER=1, MST_TAIL=0, MST_GIANT_BITS=1),
         dict(MST_FILTER=0, MST_TAIL=0, MST_GIANT_BITS=1, MST_LAZY_ROUND1=0),
         # the light phase's pair dedup from its second round with a large table
         dict(MST_FILTER=1, MST_TAIL=0, MST_DEDUP_MIN_EDGES=0, MST_DEDUP_ACTIVE=1e9, MST_DEDUP_MIN_RATIO=1,
              MST_DEDUP_TABLE_DIV=1, MST_DEDUP_CAP_LOG2=27),
         # ranged offers with the block-per-tile staged copy (default: warp per 32 tiles)
         dict(MST_FILTER=1, MST_RANGE_MB=0.01, MST_EMIT_SPARSE=0),
         # the caller's list walked in 2 / 3 interleaved segments (default 128, lists of >= 512 tiles),
         # and front to back
         dict(MST_FILTER=1, MST_INTERLEAVE=2, MST_TAIL=0), dict(MST_FILTER=0, MST_INTERLEAVE=3, MST_TAIL=0,
                                                                MST_LAZY_ROUND1=0),
         dict(MST_FILTER=1, MST_INTERLEAVE=0)]


def _check(P, n, src, dst, w, ids, total, shards=(2, 3), modes=MODES):
    g = P.Graph(n, src, dst, w)
    for mode in modes:
        with _env(**mode):
            r = P.boruvka_gpu(g)
            assert r.mst_edges.tolist() == list(ids), f"single-GPU edge set differs from the oracle ({mode})"
            assert r.total_weight == int(total)
            a = P.boruvka_gpu_aos(n, g.to_aos())
            assert a.mst_edges.tolist() == list(ids) and a.total_weight == int(total)
    for s in shards:
        # the sharded loop, plain and with sharded Filter-Boruvka
        for f in (0, 1):
            with _env(MST_FILTER=f):
                e = P.boruvka_gpu_emulated(g, s)
            assert e.mst_edges.tolist() == list(ids), f"{s}-shard edge set differs (filter={f})"
            assert e.total_weight == int(total)


def test_small_golden_graphs(mst):
    # hand graphs of the reference tests + 200 random graphs checked against
    # brute force (tests/golden/make_golden.py)
    for name, n, src, dst, w, ids, total in small_cases():
        _check(mst, n, src, dst, w, ids, total, shards=(2,), modes=MODES[:2])


@pytest.mark.parametrize("path", golden_gen_files(), ids=lambda p: p.stem)
def test_generated_golden_graphs(mst, path):
    g = load_npz(path)
    _check(mst, int(g["n"]), g["src"], g["dst"], g["w"], g["ids"].tolist(), int(g["total"]),
           shards=(2, 3, 8))


def test_app_b_100k_presets(mst, oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    app_b = {(100_000, 3, 1003): 5_460_175_173, (100_000, 6, 1006): 5_911_779_114,
             (100_000, 9, 1009): 5_981_724_212}
    for (n, d, seed), total in app_b.items():
        src, dst, w = oracle_mod.ref_generate_graph(n, d, seed)
        k = oracle_mod.kruskal(n, src, dst, w)
        assert k.total_weight == total
        _check(mst, n, src, dst, w, k.ids.tolist(), total, shards=(4,))


def test_round1_min_table(mst, oracle_mod):
    rng = np.random.default_rng(1)
    for n, m, wmax in [(1, 0, 1), (10, 40, 5), (5000, 40000, 2**32 - 1), (100000, 300000, 1000)]:
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(0, wmax, m, dtype=np.uint64).astype(np.uint32)  # ties -> lower id
        got = mst.api.round1_min(mst.Graph(n, src, dst, w))
        assert np.array_equal(got, oracle_mod.min_edges(n, src, dst, w))


def _oracle_check(P, O, n, src, dst, w, shards=(2,)):
    k = O.kruskal(n, src, dst, w)
    _check(P, n, src, dst, w, k.ids.tolist(), k.total_weight, shards=shards)
    return k


def test_edge_cases(mst, oracle_mod):
    P, O = mst, oracle_mod
    # n = 1: empty MST, with and without self-loops
    r = P.boruvka_gpu(P.Graph(1, [], [], []))
    assert r.mst_edges.size == 0 and r.total_weight == 0
    r = P.boruvka_gpu(P.Graph(1, [0, 0], [0, 0], [5, 1]))
    assert r.mst_edges.size == 0
    # single edge, zero weight, max weight
    _oracle_check(P, O, 2, [0], [1], [0])
    _oracle_check(P, O, 2, [1, 0], [0, 1], [2**32 - 1, 2**32 - 2])
    # self-loops and parallel edges mixed in
    _oracle_check(P, O, 4, [0, 0, 1, 1, 2, 3, 3, 0], [0, 1, 0, 2, 2, 2, 0, 3],
                  [3, 9, 4, 7, 1, 8, 2, 6])
    # duplicate weights: ties broken by lower edge id (stable Kruskal)
    rng = np.random.default_rng(2)
    n, m = 3000, 20000
    src = np.concatenate([np.arange(1, n), rng.integers(0, n, m - n + 1)]).astype(np.uint32)
    dst = np.concatenate([rng.integers(0, np.arange(1, n)), rng.integers(0, n, m - n + 1)]).astype(np.uint32)
    w = rng.integers(0, 50, m).astype(np.uint32)
    k = O.kruskal(n, src, dst, w)
    for mode in MODES:
        with _env(**mode):
            r = P.boruvka_gpu(P.Graph(n, src, dst, w))
            assert r.mst_edges.tolist() == k.ids.tolist() and r.total_weight == k.total_weight
    # the sharded exchange breaks ties by global id too (plain and filtered)
    for s in (2, 3, 8):
        for f in (0, 1):
            with _env(MST_FILTER=f):
                e = P.boruvka_gpu_emulated(P.Graph(n, src, dst, w), s)
            assert e.mst_edges.tolist() == k.ids.tolist() and e.total_weight == k.total_weight
    # all weights equal (the filter pivot then splits nothing off)
    w0 = np.zeros(m, dtype=np.uint32)
    k = O.kruskal(n, src, dst, w0)
    for mode in MODES:
        with _env(**mode):
            assert P.boruvka_gpu(P.Graph(n, src, dst, w0)).mst_edges.tolist() == k.ids.tolist()
    for s in (2, 5):
        assert P.boruvka_gpu_emulated(P.Graph(n, src, dst, w0), s).mst_edges.tolist() == k.ids.tolist()
    # only self-loops are light: the light phase is empty
    sl = np.concatenate([np.arange(50, dtype=np.uint32), src])
    dl = np.concatenate([np.arange(50, dtype=np.uint32), dst])
    wl = np.concatenate([np.zeros(50, dtype=np.uint32), w + 1000])
    k = O.kruskal(n, sl, dl, wl)
    for mode in MODES:
        with _env(**mode):
            assert P.boruvka_gpu(P.Graph(n, sl, dl, wl)).mst_edges.tolist() == k.ids.tolist()


def test_disconnected_returns_forest(mst, oracle_mod):
    P, O = mst, oracle_mod
    src = np.array([0, 1, 0, 3, 4, 3], dtype=np.uint32)
    dst = np.array([1, 2, 2, 4, 5, 5], dtype=np.uint32)
    w = np.array([1, 2, 3, 4, 5, 6], dtype=np.uint32)
    for n in (6, 9):  # 9: three isolated vertices too
        for mode in MODES:
            with _env(**mode):
                with pytest.raises(P.GraphError) as ei:
                    P.boruvka_gpu(P.Graph(n, src, dst, w))
                assert ei.value.kind == "Disconnected"
                f = ei.value.forest
                assert f.mst_edges.tolist() == O.kruskal(n, src, dst, w).ids.tolist() == [0, 1, 3, 4]
        with pytest.raises(P.GraphError):
            P.boruvka_gpu_emulated(P.Graph(n, src, dst, w), 2)
    with pytest.raises(P.GraphError) as ei:
        P.boruvka_gpu(P.Graph(5, [], [], []))
    assert ei.value.kind == "Disconnected" and ei.value.forest.mst_edges.size == 0


def test_input_errors(mst):
    P = mst
    for mode in MODES:
        with _env(**mode):
            with pytest.raises(P.GraphError) as ei:
                P.boruvka_gpu(P.Graph(3, [0, 3], [1, 2], [1, 2]))
            assert ei.value.kind == "EndpointOutOfRange"
    with pytest.raises(P.GraphError) as ei:
        P.boruvka_gpu_emulated(P.Graph(3, [0, 1], [1, 7], [1, 2]), 2)
    assert ei.value.kind == "EndpointOutOfRange"
    aos = P.Graph(3, [0, 1], [1, 2], [1, 2]).to_aos()
    aos["weight"][1] = 2**32 + 5
    for mode in MODES:
        with _env(**mode):
            with pytest.raises(P.GraphError) as ei:
                P.boruvka_gpu_aos(3, aos)
            assert ei.value.kind == "WeightOverflow"


def test_adversarial_shapes(mst, oracle_mod):
    P, O = mst, oracle_mod
    n = 1_000_000
    # path with increasing weights: the hook forest is one chain of depth n
    a = np.arange(n - 1, dtype=np.uint32)
    _oracle_check(P, O, n, a, a + 1, np.arange(n - 1, dtype=np.uint32), shards=(2,))
    # and decreasing weights
    _oracle_check(P, O, n, a, a + 1, np.arange(n - 1, 0, -1, dtype=np.uint32), shards=())
    # star: one hub component absorbs everything in round 1
    _oracle_check(P, O, n, np.zeros(n - 1, dtype=np.uint32), a + 1,
                  np.random.default_rng(0).permutation(n - 1).astype(np.uint32), shards=(2,))
    # dense small graph (complete K_400) with random distinct weights
    k = 400
    iu = np.triu_indices(k, 1)
    ws = np.random.default_rng(1).permutation(iu[0].size).astype(np.uint32)
    _oracle_check(P, O, k, iu[0], iu[1], ws, shards=(3,))


def test_workspace_reuse_across_sizes(mst, oracle_mod):
    """Big, small, big, repeated: look-back epochs and grown buffers stay valid."""
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    specs = [C.uniform(200_000, 1_000_000, seed=5), C.grid(3, 4, seed=1),
             C.rmat(14, 8, seed=3), C.uniform(200_000, 1_000_000, seed=5)]
    first = None
    for spec in specs:
        g = C.generate_host(spec)
        k = O.kruskal(g.n, g.src, g.dst, g.w)
        for _ in range(2):
            r = P.boruvka_gpu(g)
            assert r.mst_edges.tolist() == k.ids.tolist() and r.total_weight == k.total_weight
        if first is None:
            first = r.mst_edges
    assert np.array_equal(first, r.mst_edges)


@pytest.mark.parametrize("cfg", ["c0", "c1", "c2"])
def test_baseline_configs_full_size(mst, oracle_mod, cfg):
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    g = C.generate_host(C.CONFIGS[cfg])
    k = O.kruskal(g.n, g.src, g.dst, g.w)
    assert k.ids.size == g.n - 1
    for mode in (MODES[0], MODES[2], MODES[5], MODES[7], MODES[8]):
        with _env(**mode):
            info = P.GpuRunInfo()
            r = P.boruvka_gpu(g, info=info)
            assert np.array_equal(r.mst_edges, k.ids.astype(np.int64)) and r.total_weight == k.total_weight
            assert info.final_components == 1 and info.rounds == r.rounds >= 1
    e = P.boruvka_gpu_emulated(g, 2)
    assert np.array_equal(e.mst_edges, r.mst_edges)


@pytest.mark.parametrize("kind", ["uniform", "rmat"])
def test_sparse_large_graphs_take_the_filter(mst, oracle_mod, kind):
    """Sparse lists of >= 24 M edges with 2.5 <= m/n < 5 run Filter-Boruvka by
    default (filter_mode's second clause): default arm = forced plain loop =
    the oracle's Kruskal, single GPU and 2 emulated shards."""
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    spec = C.uniform(1 << 23, 26 << 20, seed=9) if kind == "uniform" else C.rmat(23, 3, seed=9)
    g = C.generate_host(spec)
    assert g.src.size >= (24 << 20) and 2 * g.src.size >= 5 * g.n and g.src.size < 5 * g.n
    k = O.kruskal(g.n, g.src, g.dst, g.w)
    info = P.GpuRunInfo()
    r = P.boruvka_gpu(g, info=info)
    assert np.array_equal(r.mst_edges, k.ids.astype(np.int64)) and r.total_weight == k.total_weight
    assert info.final_components == 1
    with _env(MST_FILTER=0):
        info0 = P.GpuRunInfo()
        r0 = P.boruvka_gpu(g, info=info0)
    assert np.array_equal(r0.mst_edges, r.mst_edges) and r0.total_weight == r.total_weight
    assert info.rounds != info0.rounds or info.kernel_launches != info0.kernel_launches  # the arms differ
    e = P.boruvka_gpu_emulated(g, 2)
    assert np.array_equal(e.mst_edges, r.mst_edges) and e.total_weight == r.total_weight


def test_c3_full_size(mst, oracle_mod):
    """268 M edges from the host API: plain loop = Filter-Boruvka = the
    oracle's answer, plus the restated verify_mst's structural checks."""
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    g = C.generate_host(C.CONFIGS["c3"])
    with _env(MST_FILTER=0):
        r0 = P.boruvka_gpu(g)
    r = P.boruvka_gpu(g)
    assert np.array_equal(r.mst_edges, r0.mst_edges) and r.total_weight == r0.total_weight
    v = O.verify(g.n, g.src, g.dst, g.w, r.mst_edges.astype(np.uint32))
    assert v["edge_count_ok"] and v["is_acyclic"] and v["is_spanning"]
    assert v["total_weight"] == r.total_weight
    a = _answer("c3")  # the oracle's answer (tests/golden/make_answers.py)
    assert r.mst_edges.size == a["count"] and r.total_weight == a["total_weight"]
    assert _sha_u32(r.mst_edges) == a["ids_sha256"]
    # the sharded loop with sharded Filter-Boruvka at full size
    e = P.boruvka_gpu_emulated(g, 2)
    assert np.array_equal(e.mst_edges, r.mst_edges) and e.total_weight == r.total_weight


def _answer(cfg):
    import json
    return json.loads((GOLDEN / "answers.json").read_text())[cfg]


def _sha_u32(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4", copy=False).tobytes()).hexdigest()


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_config_against_golden_answer(mst, cfg):
    """The full BASELINE config, generated on the device, against the answer
    the pinned oracle computed once (tests/golden/make_answers.py: Kruskal of
    oracle/mst_oracle.c, cross-checked with the unchanged reference's
    kruskal_oracle where it fits in RAM): edge count, u64 total and the
    SHA-256 of the ascending ids. Single GPU (device entry and the host API's
    device-input path) and the sharded loop with 2 emulated shards."""
    import ctypes
    import torch
    from paper_2005_06913_b200 import _lib as L
    from paper_2005_06913_b200 import configs as C
    P = mst
    a = _answer(cfg)
    n, m, s, d, w = C.generate_torch(C.CONFIGS[cfg])
    assert (n, m) == (a["n"], a["m"])
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    info = P.GpuRunInfo()
    count, total = P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream, info=info)
    ids = out[:count].cpu().numpy().view(np.uint32)
    assert count == a["count"] and total == a["total_weight"], (cfg, count, total)
    assert _sha_u32(ids) == a["ids_sha256"], f"{cfg}: MST edge set differs from the oracle's"
    assert info.final_components == 1
    lib = L.lib()
    lib.mst_gpu_release_workspace()
    for shards in (2,):
        e = L.MstEdgesSoa(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), 1)
        got = np.empty(n - 1, dtype=np.uint32)
        cnt, tot = ctypes.c_uint64(), ctypes.c_uint64()
        rc = lib.mst_gpu_boruvka_emulated(ctypes.byref(e), shards, got.ctypes.data, ctypes.byref(cnt),
                                          ctypes.byref(tot), None)
        assert rc == L.MST_OK, L.last_error()
        assert cnt.value == a["count"] and tot.value == a["total_weight"]
        assert _sha_u32(got[: cnt.value]) == a["ids_sha256"], f"{cfg}: {shards}-shard edge set differs"
        lib.mst_gpu_release_workspace()
    del s, d, w, out
    torch.cuda.empty_cache()


def test_gpu_generator_matches_host(mst):
    import torch
    from paper_2005_06913_b200 import configs as C
    for spec in [C.uniform(10_000, 50_000, seed=4), C.grid(33, 65, seed=2), C.rmat(13, 16, seed=7),
                 C.CONFIGS["c1"]]:
        h = C.generate_host(spec)
        n, m, s, d, w = C.generate_torch(spec)
        assert n == h.n and m == h.edge_count()
        assert np.array_equal(s.cpu().numpy().view(np.uint32), h.src)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), h.dst)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), h.w)
        del s, d, w
        torch.cuda.empty_cache()


def test_device_resident_entry(mst, oracle_mod):
    import torch
    from paper_2005_06913_b200 import configs as C
    P = mst
    spec = C.uniform(100_000, 400_000, seed=8)
    n, m, s, d, w = C.generate_torch(spec)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    hot = {}
    info = P.GpuRunInfo()
    count, total = P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream, info=info, hot=hot)
    h = C.generate_host(spec)
    k = oracle_mod.kruskal(n, h.src, h.dst, h.w)
    assert count == n - 1 and total == k.total_weight
    assert np.array_equal(out[:count].cpu().numpy().view(np.uint32), k.ids)
    assert hot["launches"] >= 2 and hot["ms"] > 0
    assert info.alg_bytes > 12 * m


def test_nccl_rank_path_single_rank(mst, oracle_mod):
    """The one-process-per-GPU entry (mst_comm_* + mst_gpu_boruvka_rank) with a
    real NCCL communicator of one rank: exercises dlopen(libnccl), comm init,
    the per-round ncclAllReduce(min, u64) and the final slot allreduce."""
    from paper_2005_06913_b200 import configs as C
    from paper_2005_06913_b200 import dist as D
    P, O = mst, oracle_mod
    uid = D.new_unique_id()
    comm = D.RankComm(uid, 1, 0, 0)
    try:
        for spec in (C.uniform(50_000, 200_000, seed=3), C.grid(100, 100, seed=2), C.rmat(13, 8, seed=5)):
            g = C.generate_host(spec)
            k = O.kruskal(g.n, g.src, g.dst, g.w)
            r = comm.boruvka(g.n, g.edge_count(), 0, g.src, g.dst, g.w)
            assert r.mst_edges.tolist() == k.ids.tolist() and r.total_weight == k.total_weight
    finally:
        comm.close()


def test_pipelined_host_copy(mst, oracle_mod):
    """Pinned SoA host arrays on the plain loop: chunked H2D on a copy stream
    with round 1's min pass per landed chunk (run_single's pipelined path)."""
    import torch
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    for spec in (C.CONFIGS["c1"], C.uniform(3_000_000, 5_000_000, seed=9)):
        g0 = C.generate_host(spec)
        k = O.kruskal(g0.n, g0.src, g0.dst, g0.w)
        pins = [torch.empty(g0.edge_count(), dtype=torch.int32, pin_memory=True) for _ in range(3)]
        for t, arr in zip(pins, (g0.src, g0.dst, g0.w)):
            t.numpy().view(np.uint32)[:] = arr
        g = P.Graph(g0.n, *(t.numpy().view(np.uint32) for t in pins))
        for mode in (dict(MST_PIPELINE_H2D=1), dict(MST_PIPELINE_H2D=0)):
            with _env(**mode):
                for _ in range(2):  # back to back: the copies must wait for the previous call
                    info = P.GpuRunInfo()
                    r = P.boruvka_gpu(g, info=info)
                    assert np.array_equal(r.mst_edges, k.ids.astype(np.int64)) and r.total_weight == k.total_weight
                    assert info.ms_h2d > 0 and info.ms_device > 0


def _retire_cases(seed=5):
    """Graphs whose light phase retires components in several rounds (round
    kernels only, MST_TAIL=0): a light perfect matching under a heavy path
    (every component is isolated in light round 2: the phase ends on zero
    components with edges), a light star forest, and a small R-MAT."""
    rng = np.random.default_rng(seed)
    out = []
    k = 30000
    n = 2 * k
    # matching (2i, 2i+1) light, a Hamiltonian path over a permutation heavy
    perm = rng.permutation(n).astype(np.uint32)
    src = np.concatenate([np.arange(0, n, 2, dtype=np.uint32), perm[:-1]])
    dst = np.concatenate([np.arange(1, n, 2, dtype=np.uint32), perm[1:]])
    w = np.concatenate([rng.permutation(k).astype(np.uint32),
                        (np.uint32(1 << 28) + rng.permutation(n - 1).astype(np.uint32))])
    out.append(("matching", n, src, dst, w))
    # stars: 2000 centres, each with 20 light leaves; centres chained heavily
    c, leaves = 2000, 20
    n2 = c * (leaves + 1)
    centre = np.repeat(np.arange(c, dtype=np.uint32), leaves)
    leaf = (c + np.arange(c * leaves)).astype(np.uint32)
    src2 = np.concatenate([centre, np.arange(c - 1, dtype=np.uint32)])
    dst2 = np.concatenate([leaf, np.arange(1, c, dtype=np.uint32)])
    w2 = np.concatenate([rng.permutation(c * leaves).astype(np.uint32),
                         (np.uint32(1 << 29) + rng.permutation(c - 1).astype(np.uint32))])
    out.append(("stars", n2, src2, dst2, w2))
    # a light random tree over half the vertices (the light phase ends with
    # one component plus the retired other half), heavy random edges over all
    n3, half = 100000, 50000
    parent = (rng.random(half - 1) * np.arange(1, half)).astype(np.uint32)
    src3 = np.concatenate([np.arange(1, half, dtype=np.uint32), rng.integers(0, n3, 300000, dtype=np.uint32),
                           np.arange(half, n3, dtype=np.uint32)])
    dst3 = np.concatenate([parent, rng.integers(0, n3, 300000, dtype=np.uint32),
                           rng.integers(0, half, n3 - half, dtype=np.uint32)])
    keep = src3 != dst3
    src3, dst3 = src3[keep], dst3[keep]
    w3 = np.empty(src3.size, dtype=np.uint32)
    w3[: half - 1] = rng.permutation(half - 1)
    w3[half - 1:] = np.uint32(1 << 28) + rng.permutation(src3.size - (half - 1)).astype(np.uint32)
    out.append(("half_tree", n3, src3, dst3, w3))
    return out


@pytest.mark.parametrize("beta", [0.25, 0.5, 1.5])
def test_light_phase_retirement(mst, oracle_mod, beta):
    """Retirement of isolated light components (kernels.cuh "retirement"):
    same MST with and without it, equal to the oracle, for graphs whose
    light phase ends with every component retired."""
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    cases = _retire_cases()
    g = C.generate_host(C.rmat(14, 8, seed=9))
    cases.append(("rmat14", g.n, g.src, g.dst, g.w))
    for name, n, src, dst, w in cases:
        k = O.kruskal(n, src, dst, w)
        G = P.Graph(n, src, dst, w)
        for retire, tail in ((1, 0), (0, 0), (1, 1)):
            # tail on: light rounds past the round kernels run in the tail with
            # TailArgs.retired (one component left ends the light phase there)
            with _env(MST_FILTER=1, MST_TAIL=tail, MST_TAIL_EDGES=20000, MST_FILTER_BETA=beta, MST_RETIRE=retire,
                      MST_DEDUP_MIN_EDGES=0):
                r = P.boruvka_gpu(G)
                e = P.boruvka_gpu_emulated(G, 2)
            assert r.mst_edges.tolist() == k.ids.tolist(), f"{name} beta={beta} retire={retire} tail={tail}: edge set differs"
            assert r.total_weight == k.total_weight
            assert e.mst_edges.tolist() == k.ids.tolist() and e.total_weight == k.total_weight, \
                f"{name} beta={beta} retire={retire}: 2-shard edge set differs"


@pytest.mark.parametrize("mode", [dict(MST_FILTER=1, MST_TAIL=0), dict(MST_FILTER=1), dict(MST_FILTER=0)])
def test_disconnected_large_forest(mst, oracle_mod, mode):
    """Two disjoint R-MAT graphs plus isolated vertices: the minimum spanning
    forest through Filter-Boruvka with retirement (components retired in the
    light phase must stay separate trees) and the plain loop."""
    from paper_2005_06913_b200 import configs as C
    P, O = mst, oracle_mod
    g = C.generate_host(C.rmat(14, 8, seed=21))
    n1 = g.n
    src = np.concatenate([g.src, g.src + np.uint32(n1)])
    dst = np.concatenate([g.dst, g.dst + np.uint32(n1)])
    rng = np.random.default_rng(4)
    w = rng.permutation(src.size).astype(np.uint32)
    n = 2 * n1 + 1000  # 1000 isolated vertices
    k = O.kruskal(n, src, dst, w)
    with _env(**mode):
        with pytest.raises(P.GraphError) as ei:
            P.boruvka_gpu(P.Graph(n, src, dst, w))
    assert ei.value.kind == "Disconnected"
    f = ei.value.forest
    assert f.mst_edges.tolist() == k.ids.tolist() and f.total_weight == k.total_weight
