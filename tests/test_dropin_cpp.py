"""The C++ drop-in entry (include/mst/boruvka_gpu.hpp) against the reference's
own Graph / generate_graph / kruskal_oracle / verify_mst, compiled from the
unchanged reference sources (tests/cpp/test_dropin.cpp, oracle/Makefile)."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "oracle" / "_ref" / "test_dropin"


def _need_bin():
    if not BIN.exists():
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")


def test_dropin_cpu_contract():
    """num_gpus < 1 -> std::invalid_argument; no device -> WorkerPanic."""
    _need_bin()
    from paper_2005_06913_b200 import _lib as L
    if L.lib().mst_gpu_device_count() > 0:
        pytest.skip("a GPU is present; the full suite covers this")
    r = subprocess.run([str(BIN), "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_full():
    _need_bin()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
