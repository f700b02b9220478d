"""The C-ABI library: loads, exports every declared symbol, validates
arguments before touching a device (CPU only)."""
import ctypes

import numpy as np
import pytest

from paper_2005_06913_b200 import _lib as L
from paper_2005_06913_b200 import api


@pytest.fixture(scope="module")
def lib():
    from paper_2005_06913_b200.build import build_library
    build_library(verbose=False)
    return L.lib()


def test_exports_every_header_symbol(lib):
    names = L.header_functions()
    assert len(names) >= 15, names
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/mst_gpu.h but not exported"
        assert name in L._SIGNATURES, f"{name} has no ctypes signature"


def test_header_struct_sizes_match_reference_layout():
    # mst::Edge is 16 bytes (graph.hpp:41-45); the AoS entry takes it as is.
    assert ctypes.sizeof(L.MstEdge) == 16
    assert api.EDGE_DTYPE.itemsize == 16


def test_version_and_device_count(lib):
    assert b"sm_100a" in lib.mst_gpu_version()
    assert lib.mst_gpu_device_count() >= 0


def _soa(n, m, on_device=0, null=False):
    p = 0 if null else 16
    return L.MstEdgesSoa(n, m, p, p, p, on_device)


def test_invalid_arguments_are_rejected_before_device_work(lib):
    ids = np.zeros(4, dtype=np.uint32)
    cnt, tot = ctypes.c_uint64(), ctypes.c_uint64()
    st = L.MstStats()
    # n < 1 (graph.cpp:93)
    e = _soa(0, 0)
    assert lib.mst_gpu_boruvka(ctypes.byref(e), 1, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    assert "vertex count" in L.last_error()
    # m too large for 32-bit edge ids
    e = _soa(5, 0xFFFFFFFF)
    assert lib.mst_gpu_boruvka(ctypes.byref(e), 1, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    # num_gpus outside [1, 8] (num_workers < 1 -> invalid_argument, boruvka_parallel.cpp:86)
    e = _soa(5, 3)
    for g in (0, -2, 9):
        assert lib.mst_gpu_boruvka(ctypes.byref(e), g, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    # NULL edge arrays with m > 0
    e = _soa(5, 3, null=True)
    assert lib.mst_gpu_boruvka(ctypes.byref(e), 1, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    # NULL output with n > 1
    e = _soa(5, 3)
    assert lib.mst_gpu_boruvka(ctypes.byref(e), 1, None, ctypes.byref(cnt), ctypes.byref(tot),
                               ctypes.byref(st)) == L.MST_ERR_INVALID_ARG
    # device input needs a single GPU
    e = _soa(5, 3, on_device=1)
    assert lib.mst_gpu_boruvka(ctypes.byref(e), 2, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    # emulated shards bound
    e = _soa(5, 3)
    assert lib.mst_gpu_boruvka_emulated(ctypes.byref(e), 0, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    assert lib.mst_gpu_boruvka_aos(0, 0, None, 0, ids.ctypes.data, None, None, None) == L.MST_ERR_INVALID_ARG
    assert lib.mst_comm_init(None, 1, 0, 0, None) == L.MST_ERR_INVALID_ARG
    assert lib.mst_comm_destroy(None) == L.MST_OK


def test_python_api_maps_errors(lib):
    g = api.build_graph(3, [(0, 1, 1), (1, 2, 2)])
    with pytest.raises(ValueError):
        api.boruvka_gpu(g, num_gpus=0)  # boruvka_parallel.cpp:86 analogue
    with pytest.raises(ValueError):
        api.build_graph(0, [])
    with pytest.raises(api.GraphError):
        api.Graph(2, [0], [1], [2**32])  # weight does not fit the device key


def test_no_device_is_loud(lib):
    if lib.mst_gpu_device_count() > 0:
        pytest.skip("a GPU is present")
    g = api.build_graph(3, [(0, 1, 1), (1, 2, 2)])
    with pytest.raises(api.WorkerPanic, match="no CUDA device"):
        api.boruvka_gpu(g)


def test_generator_validation(lib):
    from paper_2005_06913_b200 import configs as C
    with pytest.raises(ValueError):
        C.edge_count(C.uniform(1, 0, seed=0))
    with pytest.raises(ValueError):
        C.edge_count(C.uniform(10, 5, seed=0))  # m < n-1 cannot connect
    with pytest.raises(ValueError):
        C.edge_count(C.GenSpec(kind=7))


def test_tuning_table(lib):
    """Every engine knob sits in one table set through the ABI (the library
    never reads the environment)."""
    names = api.tuning_names()
    assert "MST_FILTER" in names and "MST_TAIL" in names and len(names) == len(set(names))
    beta = api.get_tuning("MST_FILTER_BETA")  # the library's default
    assert 0.5 <= beta <= 4
    with api.tuning(MST_FILTER_BETA=0.25, MST_TAIL=0):
        assert api.get_tuning("MST_FILTER_BETA") == 0.25 and api.get_tuning("MST_TAIL") == 0
    assert api.get_tuning("MST_FILTER_BETA") == beta and api.get_tuning("MST_TAIL") == 1
    with pytest.raises(ValueError, match="unknown tuning knob"):
        api.set_tuning("MST_NO_SUCH_KNOB", 1)
    applied = api.tuning_from_env({"MST_TAIL_TINY": "0", "PATH": "/bin"})
    assert applied == {"MST_TAIL_TINY": 0.0} and api.get_tuning("MST_TAIL_TINY") == 0
    lib.mst_gpu_reset_tuning()
    assert api.get_tuning("MST_TAIL_TINY") == 1
    import subprocess
    out = subprocess.run(["grep", "-c", "getenv", str(L.PKG_DIR / "csrc" / "boruvka.cu")], capture_output=True, text=True)
    assert out.stdout.strip() == "0", "the engine must not read the environment"
