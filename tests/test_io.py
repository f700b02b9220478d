"""Edge-list files (csrc/io.cu).

* text: our parallel loader reads the reference's own save_graph output
  into exactly the reference's load_graph edges, our writer produces
  byte-identical files, and malformed files fail (or pass) exactly where
  load_graph does, with its messages (graph.cpp:228-295);
* binary SoA: host round trip here, device streaming under -m gpu.
"""
import numpy as np
import pytest

import paper_2005_06913_b200 as P


def _rand_graph(n=5000, m=40000, seed=0):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    w = rng.integers(0, 2**32, m, dtype=np.uint64).astype(np.uint32)
    return P.Graph(n, src, dst, w)


def _same(a, b):
    assert a.n == b.n
    assert np.array_equal(a.src, b.src) and np.array_equal(a.dst, b.dst) and np.array_equal(a.w, b.w)


def test_text_round_trip_and_format(tmp_path):
    g = _rand_graph()
    p = tmp_path / "g.txt"
    P.save_graph(g, p)
    want = f"{g.n} {g.edge_count()}\n" + "".join(
        f"{s} {d} {w}\n" for s, d, w in zip(g.src.tolist(), g.dst.tolist(), g.w.tolist()))
    assert p.read_text() == want  # save_graph's "%u %u %llu\n"
    _same(P.load_graph(p), g)


def test_binary_round_trip(tmp_path):
    g = _rand_graph(seed=1)
    p = tmp_path / "g.mstb"
    P.save_graph(g, p, binary=True)
    raw = p.read_bytes()
    assert raw[:8] == b"MSTSOA01" and len(raw) % 4096 == (g.edge_count() * 4) % 4096
    _same(P.load_graph(p), g)
    # empty edge list
    e = P.Graph(1, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    P.save_graph(e, tmp_path / "e.mstb", binary=True)
    _same(P.load_graph(tmp_path / "e.mstb"), e)
    P.save_graph(e, tmp_path / "e.txt")
    _same(P.load_graph(tmp_path / "e.txt"), e)


def test_binary_rejects_truncated(tmp_path):
    g = _rand_graph(seed=2)
    p = tmp_path / "g.mstb"
    P.save_graph(g, p, binary=True)
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(P.GraphError, match="truncated"):
        P.load_graph(p)


def test_reads_reference_save_graph(tmp_path, oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, d, seed in [(3000, 6, 2), (20000, 9, 7)]:
        p = tmp_path / f"ref_{n}.txt"
        oracle_mod.ref_save_generated(n, d, seed, p)
        rc, msg, rn, rs, rd, rw = oracle_mod.ref_load_graph(p)
        assert rc == 0, msg
        g = P.load_graph(p)
        assert g.n == rn
        assert np.array_equal(g.src, rs) and np.array_equal(g.dst, rd)
        assert np.array_equal(g.w.astype(np.uint64), rw)
        # our writer reproduces the reference's file byte for byte
        q = tmp_path / f"ours_{n}.txt"
        P.save_graph(g, q)
        assert q.read_bytes() == p.read_bytes()


# (file body, note). Edge lists that parse are a valid simple connected
# graph, so the reference's build_graph accepts them too.
MALFORMED = [
    ("", "empty file"),
    ("3\n", "header with one field"),
    ("3 2 1\n0 1 5\n1 2 6\n", "header with three fields"),
    ("0 0\n", "zero vertices"),
    ("4294967296 0\n", "vertex count overflow"),
    ("3 2\n0 1 5\n", "one edge line missing"),
    ("3 2\n0 1 5\n1 2\n", "two fields"),
    ("3 2\n0 1 5\n1 2 6 7\n", "four fields"),
    ("3 2\n0 1 5\n1 x 6\n", "not a number"),
    ("3 2\n0 1 5\n1 -2 6\n", "negative"),
    ("3 2\n0 1 5\n1 2 6\n0 2 7\n", "trailing edge line"),
    ("3 2\n0 1 5\n1 2 6\n\n  \n", "trailing blank lines"),
    ("3 2\r\n0 1 5\r\n1 2 6\r\n", "CRLF"),
    ("3 2\n  0   1 5  \n1 2 6", "extra spaces, no final newline"),
    ("3 2\n0\t1 5\n1 2 6\n", "tab separator"),
    ("3 2\n0 4294967296 5\n1 2 6\n", "vertex id overflow"),
    ("3 2\n0 1 18446744073709551616\n1 2 6\n", "weight overflows u64"),
    ("3 2\n\n0 1 5\n", "blank edge line"),
]


@pytest.mark.parametrize("body,note", MALFORMED, ids=[n for _, n in MALFORMED])
def test_parse_rules_match_reference(tmp_path, oracle_mod, body, note):
    p = tmp_path / "f.txt"
    p.write_bytes(body.encode())
    try:
        g = P.load_graph(p)
        ours = 0
    except P.GraphError as e:
        assert e.kind == "ParseError", note
        ours, our_msg = 1, str(e).split(": ", 1)[1]
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    rc, msg, rn, rs, rd, rw = oracle_mod.ref_load_graph(p)
    assert ours == rc, (note, msg)
    if rc == 1:
        assert our_msg == msg.split(": ", 1)[1], note  # load_graph's detail text
    else:
        assert g.n == rn and np.array_equal(g.src, rs) and np.array_equal(g.w.astype(np.uint64), rw)


def test_weight_beyond_32_bits(tmp_path):
    p = tmp_path / "w.txt"
    p.write_text("2 1\n0 1 4294967296\n")
    with pytest.raises(P.GraphError, match="WeightOverflow"):
        P.load_graph(p)


def test_large_text_parallel(tmp_path):
    # many chunks: the parallel split must keep line order
    g = _rand_graph(n=100_000, m=2_000_000, seed=3)
    p = tmp_path / "big.txt"
    P.save_graph(g, p)
    _same(P.load_graph(p), g)


@pytest.mark.gpu
def test_binary_to_device(tmp_path):
    import torch
    from paper_2005_06913_b200 import configs as C
    g = C.generate_host(C.CONFIGS["c1"])
    p = tmp_path / "c1.mstb"
    P.save_graph(g, p, binary=True)
    n, m, s, d, w = P.load_graph_device(p)
    assert n == g.n and m == g.edge_count()
    assert np.array_equal(s.cpu().numpy().view(np.uint32), g.src)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), g.dst)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), g.w)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt, total = P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream)
    r = P.boruvka_gpu(g)
    assert cnt == r.mst_edges.size and total == r.total_weight
    assert np.array_equal(out[:cnt].cpu().numpy().view(np.uint32), r.mst_edges)
