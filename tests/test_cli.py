"""mstbench_gpu: the reference's benchmark CLI (proj/tools/mstbench.cpp,
run_bench bench.cpp:89-147, CSV bench.cpp:159-166) re-hosted for the GPU
path — subcommands, CSV schema, exit codes (0 ok, 1 usage, 2 graph error,
3 verification failure / worker panic)."""
import csv
import subprocess
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
    assert r.returncode == 0 and "2.5000" in r.stdout
    p.write_text("not,a,csv\n")
    assert run(cli, "summarize", "--csv", p).returncode == 1


@pytest.mark.gpu
def test_run_verify_csv(cli, tmp_path):
    out = tmp_path / "c1.csv"
    r = run(cli, "run", "--config", "c1", "--algo", "gpu,gpu-device", "--reps", "2", "--verify", "--csv", out)
    assert r.returncode == 0, r.stderr
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
