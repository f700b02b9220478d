"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the CPU checkers:
  * liboracle.so  — plain-C restatement (mst_oracle.c), always built;
  * _ref/libmstref.so — the unchanged reference library (+ ref_adapter.cpp),
    built only where /root/reference exists, then shipped with the repo.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module. The product path never does.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmstref.so"

_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)

_oracle = None
_ref = None

ALGO_KRUSKAL, ALGO_SEQ, ALGO_SEQ_OPT, ALGO_CAS, ALGO_LOCK = range(5)


@dataclass
class OracleResult:
    ids: np.ndarray        # ascending uint32 edge ids
    total_weight: int
    rounds: int = 1
    elapsed_ms: float = 0.0
    m_prime: int = 0       # reference adapter: edges fed to build_graph


def _load_oracle():
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = ctypes.CDLL(str(ORACLE_SO))
        lib.oracle_kruskal.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp, _u64p, _u64p]
        lib.oracle_boruvka_seq.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp, _u64p, _u64p, _u32p]
        lib.oracle_min_edges.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp]
        lib.oracle_verify.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp, _u64, _u32p, _u64p]
        gen_args = [ctypes.c_int, _u32, _u64, _u32, _u32, _u32, _u32, ctypes.c_double, ctypes.c_double,
                    ctypes.c_double, _u64, ctypes.c_int]
        lib.oracle_gen_count.argtypes = gen_args + [_u64p]
        lib.oracle_gen.argtypes = gen_args + [_vp, _vp, _vp, _u64p]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def _load_ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing: build with `make -C oracle ref` where "
                               "/root/reference exists")
        lib = ctypes.CDLL(str(REF_SO))
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_generate_graph.argtypes = [_u32, ctypes.c_int, _u64, _vp, _vp, _vp, _u64p]
        lib.ref_solve.argtypes = [ctypes.c_int, ctypes.c_int, _u32, _u64, _vp, _vp, _vp, _vp,
                                  _u64p, _u64p, ctypes.POINTER(ctypes.c_double), _u32p, _u64p]
        if hasattr(lib, "ref_prepare"):  # (a library built before the split has ref_solve only)
            lib.ref_prepare.restype = ctypes.c_void_p
            lib.ref_prepare.argtypes = [_u32, _u64, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_int)]
            lib.ref_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _vp, _u64p, _u64p,
                                    ctypes.POINTER(ctypes.c_double), _u32p, _u64p]
            lib.ref_release.argtypes = [ctypes.c_void_p]
        lib.ref_save_generated.argtypes = [_u32, ctypes.c_int, _u64, ctypes.c_char_p]
        lib.ref_load_graph.argtypes = [ctypes.c_char_p, _u32p, _u64p, _vp, _vp, _vp, _u64]
        _ref = lib
    return _ref


def _arrs(src, dst, w):
    return (np.ascontiguousarray(src, dtype=np.uint32), np.ascontiguousarray(dst, dtype=np.uint32),
            np.ascontiguousarray(w, dtype=np.uint32))


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def kruskal(n: int, src, dst, w) -> OracleResult:
    """Restated Kruskal oracle (boruvka_seq.cpp:121-143)."""
    src, dst, w = _arrs(src, dst, w)
    ids = np.empty(max(n - 1, 1), dtype=np.uint32)
    cnt, tot = ctypes.c_uint64(), ctypes.c_uint64()
    rc = _load_oracle().oracle_kruskal(n, src.size, _p(src), _p(dst), _p(w), _p(ids),
                                       ctypes.byref(cnt), ctypes.byref(tot))
    if rc:
        raise ValueError(f"oracle_kruskal failed with status {rc}")
    return OracleResult(ids[: cnt.value].copy(), int(tot.value))


def boruvka_seq(n: int, src, dst, w) -> OracleResult:
    """Restated sequential Boruvka (boruvka_seq.cpp:34-71)."""
    src, dst, w = _arrs(src, dst, w)
    ids = np.empty(max(n - 1, 1), dtype=np.uint32)
    cnt, tot, rounds = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint32()
    rc = _load_oracle().oracle_boruvka_seq(n, src.size, _p(src), _p(dst), _p(w), _p(ids),
                                           ctypes.byref(cnt), ctypes.byref(tot), ctypes.byref(rounds))
    if rc:
        raise ValueError(f"oracle_boruvka_seq failed with status {rc}")
    return OracleResult(ids[: cnt.value].copy(), int(tot.value), int(rounds.value))


def min_edges(n: int, src, dst, w) -> np.ndarray:
    """Round-1 lightest-edge key per vertex (boruvka_seq.cpp:47-56)."""
    src, dst, w = _arrs(src, dst, w)
    out = np.empty(n, dtype=np.uint64)
    rc = _load_oracle().oracle_min_edges(n, src.size, _p(src), _p(dst), _p(w), _p(out))
    if rc:
        raise ValueError(f"oracle_min_edges failed with status {rc}")
    return out


def verify(n: int, src, dst, w, ids) -> dict:
    """Structural checks of verify_mst (verify.cpp:15-57)."""
    src, dst, w = _arrs(src, dst, w)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    flags, total = ctypes.c_uint32(), ctypes.c_uint64()
    rc = _load_oracle().oracle_verify(n, src.size, _p(src), _p(dst), _p(w), _p(ids), ids.size,
                                      ctypes.byref(flags), ctypes.byref(total))
    if rc:
        raise IndexError("verify: edge id out of range")
    f = flags.value
    return {"edge_count_ok": bool(f & 1), "is_acyclic": bool(f & 2), "is_spanning": bool(f & 4),
            "total_weight": int(total.value)}


RMAT_ABC = (0.57, 0.19, 0.19)


def _gen_args(spec, threads: int):
    """spec: a paper_2005_06913_b200.configs.GenSpec (plain data; nothing of
    the product library is loaded) or any object with the same fields."""
    a, b, c = RMAT_ABC
    n = spec.n
    if spec.kind == 1:
        n = spec.rows * spec.cols
    elif spec.kind == 2:
        n = 1 << spec.scale
    return [spec.kind, n, spec.m, spec.rows, spec.cols, spec.scale, spec.edgefactor, a, b, c, spec.seed, threads]


def gen_count(spec, threads: int = 0) -> int:
    """Edge count of a seeded BASELINE-config graph (gen_oracle.c)."""
    out = ctypes.c_uint64()
    rc = _load_oracle().oracle_gen_count(*_gen_args(spec, threads), ctypes.byref(out))
    if rc:
        raise ValueError(f"oracle_gen_count failed with status {rc}")
    return int(out.value)


def generate(spec, threads: int = 0):
    """(n, src, dst, w) of a seeded BASELINE-config graph, built by the
    restated generator (gen_oracle.c) without the product library: the
    same bytes as configs.generate_host / generate_device."""
    m = gen_count(spec, threads)
    src, dst, w = (np.empty(m, dtype=np.uint32) for _ in range(3))
    out = ctypes.c_uint64()
    rc = _load_oracle().oracle_gen(*_gen_args(spec, threads), _p(src), _p(dst), _p(w), ctypes.byref(out))
    if rc or out.value != m:
        raise ValueError(f"oracle_gen failed with status {rc}")
    n = _gen_args(spec, threads)[1]
    return n, src, dst, w


def ref_generate_graph(n: int, avg_degree: int, seed: int):
    """The reference's own generate_graph (graph.cpp:143-194), unchanged."""
    lib = _load_ref()
    m = n * avg_degree // 2
    src, dst, w = (np.empty(m, dtype=np.uint32) for _ in range(3))
    mm = ctypes.c_uint64()
    rc = lib.ref_generate_graph(n, avg_degree, seed, _p(src), _p(dst), _p(w), ctypes.byref(mm))
    if rc:
        raise ValueError(lib.ref_last_error().decode())
    return src, dst, w


def ref_save_generated(n: int, avg_degree: int, seed: int, path) -> None:
    """The reference's save_graph(generate_graph(n, deg, seed), path)."""
    lib = _load_ref()
    if lib.ref_save_generated(n, avg_degree, seed, str(path).encode()):
        raise OSError(lib.ref_last_error().decode())


def ref_load_graph(path, cap: int = 1 << 22):
    """The reference's load_graph(path): (status, message, n, src, dst, w);
    status 0 ok, 1 ParseError, 2 other GraphError, 3 other exception."""
    lib = _load_ref()
    n, m = ctypes.c_uint32(0), ctypes.c_uint64(0)
    src, dst = np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
    w = np.zeros(cap, np.uint64)
    rc = lib.ref_load_graph(str(path).encode(), ctypes.byref(n), ctypes.byref(m), _p(src), _p(dst), _p(w), cap)
    k = min(int(m.value), cap)
    return rc, lib.ref_last_error().decode(), int(n.value), src[:k], dst[:k], w[:k]


def ref_solve(n: int, src, dst, w, algo: int = ALGO_KRUSKAL, threads: int = 1) -> OracleResult:
    """Run the unchanged reference algorithm through the §8(c) adapter."""
    lib = _load_ref()
    src, dst, w = _arrs(src, dst, w)
    ids = np.empty(max(n - 1, 1), dtype=np.uint32)
    cnt, tot, mp = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    ms, rounds = ctypes.c_double(), ctypes.c_uint32()
    rc = lib.ref_solve(algo, threads, n, src.size, _p(src), _p(dst), _p(w), _p(ids),
                       ctypes.byref(cnt), ctypes.byref(tot), ctypes.byref(ms), ctypes.byref(rounds),
                       ctypes.byref(mp))
    if rc:
        raise ValueError(f"ref_solve status {rc}: {lib.ref_last_error().decode()}")
    return OracleResult(ids[: cnt.value].copy(), int(tot.value), int(rounds.value), float(ms.value),
                        int(mp.value))


class RefGraph:
    """One input list through the §8(c) adapter, built once (sort, collapse,
    the reference's build_graph) and solved any number of times by the
    unchanged reference algorithms: the CPU legs of bench.py time several runs
    of one sample, and the adapter is not part of any of them."""

    def __init__(self, n: int, src, dst, w):
        self._lib = _load_ref()
        self.n = int(n)
        self._h = None
        self._arrays = None
        if not hasattr(self._lib, "ref_prepare"):
            self._arrays = _arrs(src, dst, w)  # old library: every solve re-runs the adapter
            return
        src, dst, w = _arrs(src, dst, w)
        st = ctypes.c_int(0)
        self._h = self._lib.ref_prepare(self.n, src.size, _p(src), _p(dst), _p(w), ctypes.byref(st))
        if not self._h:
            raise ValueError(f"ref_prepare status {st.value}: {self._lib.ref_last_error().decode()}")

    def solve(self, algo: int = ALGO_KRUSKAL, threads: int = 1) -> OracleResult:
        if self._h is None:
            return ref_solve(self.n, *self._arrays, algo, threads)
        ids = np.empty(max(self.n - 1, 1), dtype=np.uint32)
        cnt, tot, mp = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        ms, rounds = ctypes.c_double(), ctypes.c_uint32()
        rc = self._lib.ref_run(self._h, algo, threads, _p(ids), ctypes.byref(cnt), ctypes.byref(tot),
                               ctypes.byref(ms), ctypes.byref(rounds), ctypes.byref(mp))
        if rc:
            raise ValueError(f"ref_run status {rc}: {self._lib.ref_last_error().decode()}")
        return OracleResult(ids[: cnt.value].copy(), int(tot.value), int(rounds.value), float(ms.value),
                            int(mp.value))

    def close(self) -> None:
        if self._h:
            self._lib.ref_release(self._h)
            self._h = None

    def __del__(self):
        self.close()


def omp_max_threads() -> int:
    """omp_get_max_threads() inside the reference library (mstbench.cpp:137-138)."""
    if ref_available():
        return int(_load_ref().ref_omp_max_threads())
    import os
    return os.cpu_count() or 1


def hardware_threads() -> int:
    if ref_available():
        return int(_load_ref().ref_hardware_threads())
    import os
    return os.cpu_count() or 1
