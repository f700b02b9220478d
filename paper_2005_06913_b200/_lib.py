"""ctypes binding of the C ABI declared in include/mst_gpu.h.

The CUDA library is built in-tree (``paper_2005_06913_b200/libmstgpu.so``,
see build.py). There is no CPU fallback: if the library is missing, every
entry point raises ``RuntimeError`` loudly.
"""
from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_ROOT = PKG_DIR.parent
# MST_GPU_LIB: another build of the same library (A/B timing of two
# versions in tools/, e.g. tools/ab/); the product path is the in-tree one
LIB_PATH = Path(os.environ["MST_GPU_LIB"]) if os.environ.get("MST_GPU_LIB") else PKG_DIR / "libmstgpu.so"
HEADER = REPO_ROOT / "include" / "mst_gpu.h"

MST_OK = 0
MST_ERR_INVALID_ARG = 1
MST_ERR_RANGE = 2
MST_ERR_WEIGHT = 3
MST_ERR_DISCONNECTED = 4
MST_ERR_CUDA = 5
MST_ERR_NCCL = 6
MST_ERR_NO_DEVICE = 7
MST_ERR_OOM = 8
MST_ERR_STALL = 9
MST_ERR_PARSE = 10
MST_ERR_IO = 11
MST_MAX_ROUNDS = 48
MST_UNIQUE_ID_BYTES = 128

u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)


class MstEdgesSoa(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint32),
        ("m", ctypes.c_uint64),
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("w", ctypes.c_void_p),
        ("on_device", ctypes.c_int),
    ]


class MstEdge(ctypes.Structure):
    """The reference's ``mst::Edge`` (graph.hpp:41-45), 16 bytes."""

    _fields_ = [("src", ctypes.c_uint32), ("dest", ctypes.c_uint32), ("weight", ctypes.c_uint64)]


class MstStats(ctypes.Structure):
    _fields_ = [
        ("rounds", ctypes.c_uint32),
        ("final_components", ctypes.c_uint32),
        ("ms_total", ctypes.c_double),
        ("ms_device", ctypes.c_double),
        ("ms_h2d", ctypes.c_double),
        ("ms_d2h", ctypes.c_double),
        ("alg_bytes", ctypes.c_uint64),
        ("live_edges", ctypes.c_uint64 * MST_MAX_ROUNDS),
        ("live_comps", ctypes.c_uint64 * MST_MAX_ROUNDS),
        ("kernel_launches", ctypes.c_uint32),
        ("hot_bytes", ctypes.c_uint64),
    ]


class MstGenSpec(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("n", ctypes.c_uint32),
        ("m", ctypes.c_uint64),
        ("rows", ctypes.c_uint32),
        ("cols", ctypes.c_uint32),
        ("scale", ctypes.c_uint32),
        ("edgefactor", ctypes.c_uint32),
        ("a", ctypes.c_double),
        ("b", ctypes.c_double),
        ("c", ctypes.c_double),
        ("seed", ctypes.c_uint64),
    ]


class MstVerify(ctypes.Structure):
    _fields_ = [
        ("is_spanning", ctypes.c_int),
        ("is_acyclic", ctypes.c_int),
        ("edge_count_ok", ctypes.c_int),
        ("weight_matches_oracle", ctypes.c_int),
        ("edge_set_matches_oracle", ctypes.c_int),
        ("components", ctypes.c_uint64),
        ("weight", ctypes.c_uint64),
    ]


MST_VERIFY_NO_ORACLE = (1 << 64) - 1

MST_DTYPE_U32, MST_DTYPE_U64 = 0, 1
MST_OP_MIN, MST_OP_SUM = 0, 1
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                                ctypes.c_int)


class MstCollective(ctypes.Structure):
    _fields_ = [
        ("allreduce", ALLREDUCE_FN),
        ("ctx", ctypes.c_void_p),
        ("nranks", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("device", ctypes.c_int),
    ]

_SIGNATURES = {
    "mst_gpu_boruvka": (ctypes.c_int, [ctypes.POINTER(MstEdgesSoa), ctypes.c_int, ctypes.c_void_p,
                                       u64p, u64p, ctypes.POINTER(MstStats)]),
    "mst_gpu_boruvka_aos": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_void_p, u64p, u64p,
                                           ctypes.POINTER(MstStats)]),
    "mst_gpu_boruvka_emulated": (ctypes.c_int, [ctypes.POINTER(MstEdgesSoa), ctypes.c_int,
                                                ctypes.c_void_p, u64p, u64p,
                                                ctypes.POINTER(MstStats)]),
    "mst_comm_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "mst_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_void_p)]),
    "mst_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "mst_gpu_boruvka_rank": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                            ctypes.c_void_p, u64p, u64p,
                                            ctypes.POINTER(MstStats)]),
    "mst_gpu_boruvka_rank_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                                   ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_void_p, u64p, u64p, ctypes.POINTER(MstStats)]),
    "mst_gpu_boruvka_rank_cb": (ctypes.c_int, [ctypes.POINTER(MstCollective), ctypes.c_uint32, ctypes.c_uint64,
                                               ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                               ctypes.c_void_p, u64p, u64p, ctypes.POINTER(MstStats)]),
    "mst_gpu_boruvka_device": (ctypes.c_int, [ctypes.POINTER(MstEdgesSoa), ctypes.c_void_p,
                                              ctypes.c_void_p, u64p, u64p,
                                              ctypes.POINTER(MstStats),
                                              ctypes.POINTER(ctypes.c_double), u32p]),
    "mst_gpu_round1_min": (ctypes.c_int, [ctypes.POINTER(MstEdgesSoa), ctypes.c_void_p]),
    "mst_gpu_verify": (ctypes.c_int, [ctypes.POINTER(MstEdgesSoa), ctypes.c_void_p, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.POINTER(MstVerify)]),
    "mst_gpu_verify_aos": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(MstVerify)]),
    "mst_io_text_header": (ctypes.c_int, [ctypes.c_char_p, u32p, u64p]),
    "mst_io_load_text": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "mst_io_save_text": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "mst_io_soa_header": (ctypes.c_int, [ctypes.c_char_p, u32p, u64p]),
    "mst_io_load_soa": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "mst_io_save_soa": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "mst_gpu_set_tuning": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_double]),
    "mst_gpu_get_tuning": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]),
    "mst_gpu_reset_tuning": (ctypes.c_int, []),
    "mst_gpu_tuning_name": (ctypes.c_char_p, [ctypes.c_int]),
    "mst_gpu_release_workspace": (ctypes.c_int, []),
    "mst_gpu_last_error": (ctypes.c_char_p, []),
    "mst_gpu_version": (ctypes.c_char_p, []),
    "mst_gpu_device_count": (ctypes.c_int, []),
    "mst_gen_count": (ctypes.c_int, [ctypes.POINTER(MstGenSpec), u64p]),
    "mst_gen_host": (ctypes.c_int, [ctypes.POINTER(MstGenSpec), ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_int]),
    "mst_gen_device": (ctypes.c_int, [ctypes.POINTER(MstGenSpec), ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]),
}

_lib = None


def header_functions() -> list[str]:
    """Every function the C header declares (for the export test)."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w ]+?\*?\s*\b(mst_\w+)\s*\(", text, flags=re.M)))


def lib() -> ctypes.CDLL:
    """The loaded CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the MST path)")
        handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().mst_gpu_last_error().decode()
