"""mstbench_gpu: the reference's benchmark CLI (proj/tools/mstbench.cpp,
run_bench bench.cpp:89-147, CSV bench.cpp:159-166) re-hosted for the GPU
path — subcommands, CSV schema, exit codes (0 ok, 1 usage, 2 graph error,
3 verification failure / worker panic)."""
import csv
import subprocess

import numpy as np
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2005_06913_b200" / "mstbench_gpu"
HEADER = ["graph", "algorithm", "threads", "trial", "elapsed_ms", "mst_weight", "rounds", "verified"]


@pytest.fixture(scope="module")
def cli():
    from paper_2005_06913_b200.build import build_cli, build_library
    build_library(verbose=False)
    build_cli(verbose=False)
    return CLI


def run(cli, *args):
    return subprocess.run([str(cli), *map(str, args)], capture_output=True, text=True, timeout=600)


def test_presets_and_usage(cli):
    r = run(cli, "--list-presets")
    assert r.returncode == 0 and [l.split(":")[0] for l in r.stdout.splitlines()] == ["c0", "c1", "c2", "c3", "c4"]
    for bad in ([], ["bogus"], ["run", "--config", "c0", "--algo", "gpu"], ["run", "--config", "c0", "--csv", "x"],
                ["run", "--config", "c9", "--algo", "gpu", "--csv", "x"],
                ["run", "--config", "c0", "--algo", "cas", "--csv", "x"],
                ["run", "--config", "c0", "--graph", "g.txt", "--algo", "gpu", "--csv", "x"],
                ["run", "--config", "c0", "--algo", "gpu", "--reps", "0", "--csv", "x"],
                ["generate", "--config", "c0"]):
        assert run(cli, *bad).returncode == 1, bad


def test_generate_matches_library(cli, tmp_path):
    import numpy as np
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C
    out = tmp_path / "c0.mstb"
    r = run(cli, "generate", "--config", "c0", "--out", out, "--binary")
    assert r.returncode == 0, r.stderr
    g = P.load_graph(out)
    ref = C.generate_host(C.CONFIGS["c0"])
    assert g.n == ref.n and np.array_equal(g.src, ref.src) and np.array_equal(g.w, ref.w)
    txt = tmp_path / "c0.txt"
    assert run(cli, "generate", "--config", "c0", "--out", txt).returncode == 0
    with open(txt) as f:
        assert f.readline() == f"{ref.n} {ref.edge_count()}\n"


def test_graph_error_exit_code(cli, tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("3 2\n0 1 5\n")
    r = run(cli, "run", "--graph", bad, "--algo", "gpu", "--csv", tmp_path / "o.csv")
    assert r.returncode == 2 and "expected 2 edge lines" in r.stderr


def test_summarize(cli, tmp_path):
    p = tmp_path / "r.csv"
    p.write_text(",".join(HEADER) + "\ng,gpu,1,1,2.5,10,3,1\ng,gpu,1,2,1.5,10,3,1\ng,gpu,1,3,9,10,3,1\n")
    r = run(cli, "summarize", "--csv", p)
    assert r.returncode == 0 and "2.5000" in r.stdout and "vs_seq" not in r.stdout
    # the reference's own mstbench rows (seq / cas) as the baseline:
    # speedup table of bench.cpp:246-335 with the GPU rows as parallel algorithms
    b = tmp_path / "ref.csv"
    b.write_text(",".join(HEADER) + "\ng,seq,1,1,100,10,7,1\ng,seq,1,2,120,10,7,1\ng,seq,1,3,110,10,7,1\n"
                 "g,cas,4,1,50,10,9,1\ng,cas,8,1,55,10,9,1\n")
    r = run(cli, "summarize", "--csv", p, "--baseline", b)
    assert r.returncode == 0, r.stderr
    gpu = [l.split() for l in r.stdout.splitlines() if l.startswith("g ") and " gpu " in l and len(l.split()) == 6]
    assert gpu == [["g", "gpu", "1", "44.000", "-", "20.000"]], r.stdout   # 110/2.5, best cas 50/2.5
    cas4 = [l.split() for l in r.stdout.splitlines() if l.split()[:3] == ["g", "cas", "4"] and len(l.split()) == 6]
    assert cas4 == [["g", "cas", "4", "2.200", "-", "1.000"]]
    p.write_text("not,a,csv\n")
    assert run(cli, "summarize", "--csv", p).returncode == 1


def test_oracle_answer_file_roundtrip(tmp_path, oracle_mod):
    from oracle import answer as A
    ids = np.array([1, 5, 9], dtype=np.uint32)
    A.write_answer(tmp_path / "a.ans", 4, ids, 123)
    n, got, total = A.read_answer(tmp_path / "a.ans")
    assert n == 4 and total == 123 and got.tolist() == [1, 5, 9]


def test_oracle_flag_needs_verify_and_a_valid_file(cli, tmp_path):
    (tmp_path / "junk.ans").write_bytes(b"nope")
    r = run(cli, "run", "--config", "c0", "--algo", "gpu", "--oracle", tmp_path / "junk.ans", "--csv", tmp_path / "o")
    assert r.returncode == 1 and "--oracle needs --verify" in r.stderr


@pytest.mark.gpu
def test_run_verify_csv(cli, tmp_path):
    import sys
    # the oracle's answer, computed once on the CPU (oracle/answer.py), checks every trial
    ans = tmp_path / "c1.ans"
    subprocess.run([sys.executable, "-m", "oracle.answer", "--config", "c1", "--out", str(ans)], check=True, cwd=ROOT)
    out = tmp_path / "c1.csv"
    r = run(cli, "run", "--config", "c1", "--algo", "gpu,gpu-device", "--reps", "2", "--verify", "--oracle", ans,
            "--csv", out)
    assert r.returncode == 0, r.stderr
    assert "# oracle:" in r.stdout
    # a wrong answer (one id swapped) must fail verification with exit code 3
    from oracle import answer as A
    n, ids, total = A.read_answer(ans)
    bad_ids = ids.copy()
    bad_ids[0] = bad_ids[0] + 1 if bad_ids[0] + 1 not in set(ids.tolist()) else bad_ids[0] + 2
    A.write_answer(tmp_path / "bad.ans", n, np.sort(bad_ids), total)
    r2 = run(cli, "run", "--config", "c1", "--algo", "gpu", "--reps", "1", "--verify", "--oracle", tmp_path / "bad.ans",
             "--csv", tmp_path / "bad.csv")
    assert r2.returncode == 3 and "MISMATCH" in r2.stderr
    rows = list(csv.reader(open(out)))
    assert rows[0] == HEADER and len(rows) == 5
    assert {row[1] for row in rows[1:]} == {"gpu", "gpu-device"}
    assert len({row[5] for row in rows[1:]}) == 1 and all(row[7] == "1" for row in rows[1:])
    # a graph file (binary SoA) round-trips through the same loop
    g = tmp_path / "c0.mstb"
    assert run(cli, "generate", "--config", "c0", "--out", g, "--binary").returncode == 0
    r = run(cli, "run", "--graph", g, "--algo", "gpu", "--reps", "1", "--verify", "--csv", tmp_path / "c0.csv")
    assert r.returncode == 0, r.stderr
    assert "c0,gpu,T=1,trial=1:" in r.stdout
