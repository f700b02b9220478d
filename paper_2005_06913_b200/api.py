"""Python mirror of the reference's MST entry point, backed by the CUDA library.

Reference interface being replaced (one hot path, ``north_star``):

    mst::MstResult mst::boruvka_cas(mst::Graph& g, int num_workers,
                                    mst::ParallelRunInfo* info = nullptr);
    -- /root/reference/proj/include/mst/boruvka_parallel.hpp:70
       /root/reference/proj/src/boruvka_parallel.cpp:85-291

Here ``boruvka_gpu(g, num_gpus=1, info=None)`` keeps that shape: a ``Graph``
in, an ``MstResult`` out (``mst_result.hpp:15-20``: ids sorted ascending as
int64, u64 total weight, rounds, elapsed_ms), errors as exceptions with the
reference's meaning:

* ``ValueError``   ~ std::invalid_argument (num_workers < 1,
  boruvka_parallel.cpp:86; n < 1, graph.cpp:93)
* ``GraphError``   ~ mst::GraphError (graph.hpp:19-38): EndpointOutOfRange,
  Disconnected (raised after the run; ``err.forest`` holds the minimum
  spanning forest), WeightOverflow (weight >= 2^32, a device-key limit)
* ``WorkerPanic``  ~ mst::WorkerPanic (boruvka_parallel.hpp:44-47): CUDA,
  NCCL or no-progress failures.

Every call goes through the C ABI in include/mst_gpu.h; nothing falls back
to the CPU.
"""
from __future__ import annotations

import ctypes
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

__all__ = [
    "Graph", "MstResult", "GpuRunInfo", "GraphError", "WorkerPanic", "build_graph",
    "boruvka_gpu", "boruvka_gpu_aos", "boruvka_gpu_emulated", "boruvka_gpu_device",
    "VerifyReport", "verify_mst", "verify_mst_aos", "load_graph", "save_graph", "load_graph_device",
    "EDGE_DTYPE",
]

# The reference's mst::Edge {u32 src, u32 dest, u64 weight} (graph.hpp:41-45).
EDGE_DTYPE = np.dtype([("src", "<u4"), ("dest", "<u4"), ("weight", "<u8")])


class GraphError(RuntimeError):
    """Input-contract violation (mirrors mst::GraphError, graph.hpp:30-38)."""

    def __init__(self, kind: str, what: str, forest: "MstResult | None" = None):
        super().__init__(f"{kind}: {what}")
        self.kind = kind
        self.forest = forest


class WorkerPanic(RuntimeError):
    """Device/collective failure or stall (mirrors mst::WorkerPanic)."""


@dataclass
class MstResult:
    """mst::MstResult (mst_result.hpp:15-20)."""

    mst_edges: np.ndarray
    total_weight: int
    rounds: int
    elapsed_ms: float


@dataclass
class GpuRunInfo:
    """ParallelRunInfo analogue (boruvka_parallel.hpp:52-56) + round counters."""

    final_components: int = 0
    rounds: int = 0
    ms_total: float = 0.0
    ms_device: float = 0.0
    ms_h2d: float = 0.0
    ms_d2h: float = 0.0
    alg_bytes: int = 0
    live_edges: list = field(default_factory=list)
    live_comps: list = field(default_factory=list)
    kernel_launches: int = 0


class Graph:
    """Edge-list graph in the device-native SoA layout (u32 src/dst/weight).

    Mirrors mst::Graph's accessors (graph.hpp:57-60). Unlike the reference's
    build_graph, construction does not enforce the simple-graph contract:
    duplicate pairs, zero weights and self-loops are legal input to the GPU
    path (self-loops are skipped, parallel edges need no care). Endpoints are
    range-checked on the device.
    """

    def __init__(self, n: int, src, dst, w):
        self.n = int(n)
        self.src = np.ascontiguousarray(src, dtype=np.uint32)
        self.dst = np.ascontiguousarray(dst, dtype=np.uint32)
        w = np.asarray(w)
        if w.dtype != np.uint32:
            if w.size and (w.min() < 0 or w.max() > 0xFFFFFFFF):
                raise GraphError("WeightOverflow", "weights must fit in 32 bits")
            w = w.astype(np.uint32)
        self.w = np.ascontiguousarray(w)
        if not (self.src.shape == self.dst.shape == self.w.shape) or self.src.ndim != 1:
            raise ValueError("src, dst and w must be 1-D arrays of equal length")

    @classmethod
    def from_edges(cls, n: int, edges) -> "Graph":
        arr = np.asarray(list(edges), dtype=np.uint64).reshape(-1, 3)
        return cls(n, arr[:, 0], arr[:, 1], arr[:, 2])

    def vertex_count(self) -> int:
        return self.n

    def edge_count(self) -> int:
        return int(self.src.shape[0])

    def to_aos(self) -> np.ndarray:
        out = np.empty(self.edge_count(), dtype=EDGE_DTYPE)
        out["src"], out["dest"], out["weight"] = self.src, self.dst, self.w
        return out


def build_graph(n: int, edges) -> Graph:
    """Counterpart of mst::build_graph (graph.cpp:92-141) for list input."""
    if n < 1:
        raise ValueError("build_graph: vertex count must be >= 1")
    return Graph.from_edges(n, edges)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def _host_out(count: int) -> np.ndarray:
    """uint32 output buffer. When torch is already loaded, take it from torch's
    caching pinned-host allocator so the device->host copy runs at full link
    speed (16 MB: 0.3 ms pinned vs 1.1 ms pageable on the B200 host); otherwise
    plain numpy (the library stages pageable copies itself)."""
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_available():
                return torch.empty(count, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        except Exception:
            pass
    return np.empty(count, dtype=np.uint32)


def _info_from(stats: L.MstStats, info: GpuRunInfo | None) -> None:
    if info is None:
        return
    r = stats.rounds
    info.final_components = stats.final_components
    info.rounds = r
    info.ms_total = stats.ms_total
    info.ms_device = stats.ms_device
    info.ms_h2d = stats.ms_h2d
    info.ms_d2h = stats.ms_d2h
    info.alg_bytes = stats.alg_bytes
    info.live_edges = [int(stats.live_edges[i]) for i in range(min(r, L.MST_MAX_ROUNDS))]
    info.live_comps = [int(stats.live_comps[i]) for i in range(min(r, L.MST_MAX_ROUNDS))]
    info.kernel_launches = stats.kernel_launches


def _raise_for(rc: int, result: MstResult | None = None) -> None:
    if rc == L.MST_OK:
        return
    msg = L.last_error()
    if rc == L.MST_ERR_INVALID_ARG:
        raise ValueError(msg)
    if rc == L.MST_ERR_RANGE:
        raise GraphError("EndpointOutOfRange", msg)
    if rc == L.MST_ERR_WEIGHT:
        raise GraphError("WeightOverflow", msg)
    if rc == L.MST_ERR_DISCONNECTED:
        raise GraphError("Disconnected", msg, forest=result)
    if rc == L.MST_ERR_PARSE:
        raise GraphError("ParseError", msg)
    if rc == L.MST_ERR_IO:
        raise OSError(msg)
    raise WorkerPanic(f"[status {rc}] {msg}")


def _finish(rc, ids, count, total, stats, info):
    res = None
    if rc in (L.MST_OK, L.MST_ERR_DISCONNECTED):
        # uint32 ids (m < 2^32 - 1 is a boundary check); the C++ wrapper widens
        # to the reference's int64 EdgeId
        res = MstResult(ids[: count.value], int(total.value), int(stats.rounds), float(stats.ms_total))
    _info_from(stats, info)
    _raise_for(rc, res)
    return res


def boruvka_gpu(g: Graph, num_gpus: int = 1, info: GpuRunInfo | None = None) -> MstResult:
    """GPU replacement of boruvka_cas(g, num_workers, info).

    num_gpus == 1: one B200. num_gpus in 2..8: this process drives devices
    0..num_gpus-1, edge list sharded, one allreduce(min) per round.
    """
    if num_gpus < 1:
        raise ValueError("boruvka: need num_gpus >= 1")
    lib = L.lib()
    e = L.MstEdgesSoa(g.n, g.edge_count(), _ptr(g.src), _ptr(g.dst), _ptr(g.w), 0)
    ids = _host_out(max(g.n - 1, 1))
    count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
    stats = L.MstStats()
    rc = lib.mst_gpu_boruvka(ctypes.byref(e), num_gpus, ids.ctypes.data, ctypes.byref(count),
                             ctypes.byref(total), ctypes.byref(stats))
    return _finish(rc, ids, count, total, stats, info)


def boruvka_gpu_aos(n: int, edges: np.ndarray, info: GpuRunInfo | None = None) -> MstResult:
    """Same, fed the reference's AoS ``Edge`` array unchanged (EDGE_DTYPE)."""
    edges = np.ascontiguousarray(edges, dtype=EDGE_DTYPE)
    lib = L.lib()
    ids = _host_out(max(n - 1, 1))
    count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
    stats = L.MstStats()
    rc = lib.mst_gpu_boruvka_aos(n, edges.shape[0], _ptr(edges), 0, ids.ctypes.data,
                                 ctypes.byref(count), ctypes.byref(total), ctypes.byref(stats))
    return _finish(rc, ids, count, total, stats, info)


def boruvka_gpu_emulated(g: Graph, shards: int, info: GpuRunInfo | None = None) -> MstResult:
    """The multi-GPU (sharded, exchanged-key) algorithm with `shards` edge
    shards emulated on the current GPU; used to test the sharded protocol."""
    lib = L.lib()
    e = L.MstEdgesSoa(g.n, g.edge_count(), _ptr(g.src), _ptr(g.dst), _ptr(g.w), 0)
    ids = np.empty(max(g.n - 1, 1), dtype=np.uint32)
    count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
    stats = L.MstStats()
    rc = lib.mst_gpu_boruvka_emulated(ctypes.byref(e), shards, ids.ctypes.data, ctypes.byref(count),
                                      ctypes.byref(total), ctypes.byref(stats))
    return _finish(rc, ids, count, total, stats, info)


@dataclass
class VerifyReport:
    """mst::VerifyReport (verify.hpp:11-24); the oracle flags are None when
    no oracle result was given (structural checks only)."""

    is_spanning: bool
    is_acyclic: bool
    edge_count_ok: bool
    weight_matches_oracle: bool | None
    edge_set_matches_oracle: bool | None
    components: int
    weight: int
    details: str = ""

    def all_ok(self) -> bool:
        oracle = [f for f in (self.weight_matches_oracle, self.edge_set_matches_oracle) if f is not None]
        return self.is_spanning and self.is_acyclic and self.edge_count_ok and all(oracle)


def _verify_args(ids, oracle):
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= 2**32 - 1):
        raise IndexError("verify_mst: edge id outside [0, m)")
    ids = ids.astype(np.uint32)
    if oracle is None:
        return ids, np.zeros(1, dtype=np.uint32), 0, L.MST_VERIFY_NO_ORACLE
    oids = np.ascontiguousarray(oracle.mst_edges, dtype=np.int64).astype(np.uint32)
    return ids, oids, oids.size, int(oracle.total_weight)


def _report(rc, rep: "L.MstVerify", n: int, count: int, oracle, own_total) -> VerifyReport:
    if rc == L.MST_ERR_RANGE:
        raise IndexError(L.last_error())  # std::out_of_range (verify.cpp:19-22)
    _raise_for(rc)
    flag = (lambda v: None if v < 0 else bool(v))
    r = VerifyReport(bool(rep.is_spanning), bool(rep.is_acyclic), bool(rep.edge_count_ok),
                     flag(rep.weight_matches_oracle), flag(rep.edge_set_matches_oracle),
                     int(rep.components), int(rep.weight))
    # the reference's details line (verify.cpp:45-53)
    d = f"edges={count} (expected {n - 1}), weight={r.weight}"
    if oracle is not None:
        d += f" (oracle {int(oracle.total_weight)})"
    d += f", components={r.components}, acyclic={'yes' if r.is_acyclic else 'no'}"
    if r.edge_set_matches_oracle is not None:
        d += f", edge_set={'match' if r.edge_set_matches_oracle else 'MISMATCH'}"
    if own_total is not None and own_total != r.weight:
        d += f"; WARNING: result.total_weight={own_total} disagrees with its own edge list"
    r.details = d
    return r


def verify_mst(g: Graph, result: MstResult, oracle: MstResult | None = None) -> VerifyReport:
    """verify_mst(g, result, oracle) (verify.hpp:27-31) on the GPU.

    The oracle result is supplied by the caller (computed once per graph, as
    the reference's second overload does); without it only the structural
    checks run. An id outside [0, m) raises IndexError (std::out_of_range).
    """
    lib = L.lib()
    ids, oids, ocount, ototal = _verify_args(result.mst_edges, oracle)
    e = L.MstEdgesSoa(g.n, g.edge_count(), _ptr(g.src), _ptr(g.dst), _ptr(g.w), 0)
    rep = L.MstVerify()
    rc = lib.mst_gpu_verify(ctypes.byref(e), _ptr(ids), ids.size, _ptr(oids), ocount, ototal, ctypes.byref(rep))
    return _report(rc, rep, g.n, ids.size, oracle, int(result.total_weight))


def verify_mst_aos(n: int, edges: np.ndarray, result: MstResult, oracle: MstResult | None = None) -> VerifyReport:
    """Same over the reference's AoS ``Edge`` array (64-bit weights)."""
    edges = np.ascontiguousarray(edges, dtype=EDGE_DTYPE)
    lib = L.lib()
    ids, oids, ocount, ototal = _verify_args(result.mst_edges, oracle)
    rep = L.MstVerify()
    rc = lib.mst_gpu_verify_aos(n, edges.shape[0], _ptr(edges), 0, _ptr(ids), ids.size, _ptr(oids), ocount,
                                ototal, ctypes.byref(rep))
    return _report(rc, rep, n, ids.size, oracle, int(result.total_weight))


_SOA_MAGIC = b"MSTSOA01"


def _is_soa(path) -> bool:
    with open(path, "rb") as f:
        return f.read(8) == _SOA_MAGIC


def _header(path, fn) -> tuple[int, int]:
    n, m = ctypes.c_uint32(0), ctypes.c_uint64(0)
    _raise_for(fn(str(path).encode(), ctypes.byref(n), ctypes.byref(m)))
    return int(n.value), int(m.value)


def load_graph(path) -> Graph:
    """load_graph(path) (graph.cpp:228-281): the reference's text format, or
    the binary SoA format (detected by its magic). Parse errors raise
    GraphError("ParseError") with load_graph's messages."""
    lib = L.lib()
    soa = _is_soa(path)
    n, m = _header(path, lib.mst_io_soa_header if soa else lib.mst_io_text_header)
    src, dst, w = (np.empty(m, dtype=np.uint32) for _ in range(3))
    p = str(path).encode()
    if soa:
        rc = lib.mst_io_load_soa(p, n, m, _ptr(src), _ptr(dst), _ptr(w), 0)
    else:
        rc = lib.mst_io_load_text(p, n, m, _ptr(src), _ptr(dst), _ptr(w))
    _raise_for(rc)
    return Graph(n, src, dst, w)


def save_graph(g: Graph, path, binary: bool = False) -> None:
    """save_graph(g, path) (graph.cpp:283-295) in the reference's text format,
    or (binary=True) the SoA format that load_graph_device streams to HBM."""
    lib = L.lib()
    fn = lib.mst_io_save_soa if binary else lib.mst_io_save_text
    _raise_for(fn(str(path).encode(), g.n, g.edge_count(), _ptr(g.src), _ptr(g.dst), _ptr(g.w)))


def load_graph_device(path, device: int | None = None):
    """Binary SoA file -> device arrays (torch uint32-as-int32 tensors on the
    current CUDA device): returns (n, m, src, dst, w), ready for
    boruvka_gpu_device. The file is streamed through pinned chunks."""
    import torch
    lib = L.lib()
    if not _is_soa(path):
        raise GraphError("ParseError", f"{path}: not an MSTSOA01 file (use save_graph(..., binary=True))")
    n, m = _header(path, lib.mst_io_soa_header)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    src, dst, w = (torch.empty(max(m, 1), dtype=torch.int32, device=dev) for _ in range(3))
    with torch.cuda.device(dev):
        torch.cuda.synchronize()
        _raise_for(lib.mst_io_load_soa(str(path).encode(), n, m, src.data_ptr(), dst.data_ptr(), w.data_ptr(), 1))
    return n, m, src[:m], dst[:m], w[:m]


def round1_min(g: Graph) -> np.ndarray:
    """Test hook: the device's round-1 minimum table (k_min_round1 only)."""
    lib = L.lib()
    e = L.MstEdgesSoa(g.n, g.edge_count(), _ptr(g.src), _ptr(g.dst), _ptr(g.w), 0)
    out = np.empty(g.n, dtype=np.uint64)
    _raise_for(lib.mst_gpu_round1_min(ctypes.byref(e), out.ctypes.data))
    return out


def boruvka_gpu_device(n: int, m: int, src_ptr: int, dst_ptr: int, w_ptr: int, out_ptr: int,
                       stream: int = 0, info: GpuRunInfo | None = None, hot: dict | None = None):
    """Device-resident entry (edges already in HBM, ids left in HBM at out_ptr).

    Returns (count, total_weight). With ``hot`` a dict, fills
    ``hot['ms']``/``hot['launches']`` with the summed CUDA-event time and
    launch count of the edge-pass kernels (k_min_round1, k_count, k_emit).
    """
    lib = L.lib()
    e = L.MstEdgesSoa(n, m, src_ptr, dst_ptr, w_ptr, 1)
    count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
    stats = L.MstStats()
    ms_hot = ctypes.c_double(0)
    hot_n = ctypes.c_uint32(0)
    rc = lib.mst_gpu_boruvka_device(ctypes.byref(e), out_ptr, stream, ctypes.byref(count),
                                    ctypes.byref(total), ctypes.byref(stats),
                                    ctypes.byref(ms_hot) if hot is not None else None,
                                    ctypes.byref(hot_n) if hot is not None else None)
    _info_from(stats, info)
    if hot is not None:
        hot["ms"] = ms_hot.value
        hot["launches"] = hot_n.value
        hot["bytes"] = int(stats.hot_bytes)
    _raise_for(rc)
    return int(count.value), int(total.value)


# ---- tuning knobs (include/mst_gpu.h "tuning knobs") ----

def tuning_names() -> list[str]:
    """Every knob of the engine's tuning table."""
    out, i = [], 0
    while True:
        name = L.lib().mst_gpu_tuning_name(i)
        if name is None:
            return out
        out.append(name.decode())
        i += 1


def set_tuning(name: str, value: float) -> None:
    rc = L.lib().mst_gpu_set_tuning(name.encode(), float(value))
    if rc != L.MST_OK:
        raise ValueError(L.last_error())


def get_tuning(name: str) -> float:
    v = ctypes.c_double()
    rc = L.lib().mst_gpu_get_tuning(name.encode(), ctypes.byref(v))
    if rc != L.MST_OK:
        raise ValueError(L.last_error())
    return v.value


class tuning:
    """Context manager: set knobs for the calls inside, restore on exit.

        with tuning(MST_FILTER=1, MST_FILTER_BETA=0.3):
            boruvka_gpu(g)
    """

    def __init__(self, **knobs):
        self.knobs = knobs

    def __enter__(self):
        self.old = {k: get_tuning(k) for k in self.knobs}
        for k, v in self.knobs.items():
            set_tuning(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_tuning(k, v)


def tuning_from_env(environ=None) -> dict:
    """A/B tools only: reset the knobs to their defaults, then apply the
    MST_* variables of the environment that name a knob (the library itself
    never reads the environment). Returns the applied ones."""
    import os
    env = os.environ if environ is None else environ
    L.lib().mst_gpu_reset_tuning()
    applied = {}
    for name in tuning_names():
        if env.get(name):
            set_tuning(name, float(env[name]))
            applied[name] = float(env[name])
    return applied
