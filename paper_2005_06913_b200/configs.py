"""The five BASELINE.json workloads as seeded generator specs.

Seeds are the config index ("use seed = config index").
The generators (csrc/gen.cu) are counter-based, so ``generate_host`` (CPU
threads) and ``generate_device`` (CUDA) return identical bytes.

  c0  uniform, n=1,000,000,  m=4,000,000          (runs on the CPU reference)
  c1  2048 x 2048 4-neighbour grid, m=8,384,512    (high diameter)
  c2  R-MAT scale 22, edgefactor 16 (+ tree)       (skewed degrees)
  c3  uniform, n=16,777,216, m=268,435,456
  c4  R-MAT scale 26, edgefactor 16 (+ tree)       (~1.14 B edges)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .api import Graph, WorkerPanic

RMAT_ABC = (0.57, 0.19, 0.19)


@dataclass(frozen=True)
class GenSpec:
    kind: int              # 0 uniform, 1 grid, 2 rmat
    n: int = 0
    m: int = 0
    rows: int = 0
    cols: int = 0
    scale: int = 0
    edgefactor: int = 0
    seed: int = 0
    name: str = ""

    def to_c(self) -> L.MstGenSpec:
        a, b, c = RMAT_ABC
        n = self.n
        if self.kind == 1:
            n = self.rows * self.cols
        elif self.kind == 2:
            n = 1 << self.scale
        return L.MstGenSpec(self.kind, n, self.m, self.rows, self.cols, self.scale,
                            self.edgefactor, a, b, c, self.seed)

    @property
    def vertices(self) -> int:
        if self.kind == 1:
            return self.rows * self.cols
        if self.kind == 2:
            return 1 << self.scale
        return self.n


def uniform(n: int, m: int, seed: int, name: str = "") -> GenSpec:
    return GenSpec(kind=0, n=n, m=m, seed=seed, name=name or f"uniform_{n}_{m}")


def grid(rows: int, cols: int, seed: int, name: str = "") -> GenSpec:
    return GenSpec(kind=1, rows=rows, cols=cols, seed=seed, name=name or f"grid_{rows}x{cols}")


def rmat(scale: int, edgefactor: int, seed: int, name: str = "") -> GenSpec:
    return GenSpec(kind=2, scale=scale, edgefactor=edgefactor, seed=seed,
                   name=name or f"rmat_{scale}_{edgefactor}")


CONFIGS = {
    "c0": uniform(1_000_000, 4_000_000, seed=0, name="c0_uniform_1M_4M"),
    "c1": grid(2048, 2048, seed=1, name="c1_grid_2048x2048"),
    "c2": rmat(22, 16, seed=2, name="c2_rmat22_ef16"),
    "c3": uniform(16_777_216, 268_435_456, seed=3, name="c3_uniform_16.7M_268M"),
    "c4": rmat(26, 16, seed=4, name="c4_rmat26_ef16"),
}

# Edge counts of the five workloads (the R-MAT ones depend on the draws that
# land on the diagonal); pinned by tests/test_generators.py and the GPU
# golden-answer test against tests/golden/answers.json.
KNOWN_EDGES = {
    "c0_uniform_1M_4M": 4_000_000,
    "c1_grid_2048x2048": 8_384_512,
    "c2_rmat22_ef16": 71_301_337,
    "c3_uniform_16.7M_268M": 268_435_456,
    "c4_rmat26_ef16": 1_140_846_523,
}


def _check(rc: int) -> None:
    if rc != L.MST_OK:
        msg = L.last_error()
        if rc == L.MST_ERR_INVALID_ARG:
            raise ValueError(msg)
        raise WorkerPanic(f"[status {rc}] {msg}")


def edge_count(spec: GenSpec) -> int:
    out = ctypes.c_uint64(0)
    c = spec.to_c()
    _check(L.lib().mst_gen_count(ctypes.byref(c), ctypes.byref(out)))
    return int(out.value)


def generate_host(spec: GenSpec, threads: int = 0, m: int | None = None) -> Graph:
    """CPU generator (std::thread). ``m`` skips the R-MAT counting pass."""
    m = edge_count(spec) if m is None else m
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    w = np.empty(m, dtype=np.uint32)
    c = spec.to_c()
    _check(L.lib().mst_gen_host(ctypes.byref(c), src.ctypes.data, dst.ctypes.data, w.ctypes.data,
                                threads))
    return Graph(spec.vertices, src, dst, w)


def generate_device(spec: GenSpec, src_ptr: int, dst_ptr: int, w_ptr: int) -> None:
    """GPU generator into device arrays of edge_count(spec) entries."""
    c = spec.to_c()
    _check(L.lib().mst_gen_device(ctypes.byref(c), src_ptr, dst_ptr, w_ptr))


def generate_torch(spec: GenSpec, device: str = "cuda"):
    """GPU generator into fresh torch uint32... (int32 storage) tensors."""
    import torch

    m = edge_count(spec)
    src = torch.empty(m, dtype=torch.int32, device=device)
    dst = torch.empty(m, dtype=torch.int32, device=device)
    w = torch.empty(m, dtype=torch.int32, device=device)
    generate_device(spec, src.data_ptr(), dst.data_ptr(), w.data_ptr())
    return spec.vertices, m, src, dst, w
