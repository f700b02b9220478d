import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


def golden_gen_files():
    return sorted(GOLDEN.glob("gen_*.npz")) + sorted(GOLDEN.glob("multi_*.npz"))


def load_npz(path):
    z = np.load(path)
    return {k: z[k] for k in z.files}


def small_graphs():
    return json.loads((GOLDEN / "small_graphs.json").read_text())


def small_cases():
    """(name, n, src, dst, w, ids, total) for every small golden graph."""
    data = small_graphs()
    out = []
    for name, g in data.items():
        if name == "random200":
            continue
        a = np.array(g["edges"], dtype=np.uint64)
        out.append((name, g["n"], a[:, 0], a[:, 1], a[:, 2], g["ids"], g["total"]))
    for i, g in enumerate(data["random200"]):
        a = np.array(g["edges"], dtype=np.uint64)
        out.append((f"random{i}", g["n"], a[:, 0], a[:, 1], a[:, 2], g["ids"], g["total"]))
    return out


@pytest.fixture(scope="session")
def oracle_mod():
    from paper_2005_06913_b200.build import build_oracle
    from oracle import oracle as O
    if not O.ORACLE_SO.exists():
        build_oracle(verbose=False)
    return O
