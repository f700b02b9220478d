"""In-tree build of the sm_100a CUDA library (and, for tests, the oracle).

    python -m paper_2005_06913_b200.build          # library + oracle
nvcc cross-compiles for sm_100a without a GPU; the .so files are git-ignored
but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmstgpu.so"
SOURCES = ["boruvka.cu", "gen.cu", "io.cu"]
DEPS = SOURCES + ["kernels.cuh", "common.cuh", "verify.cuh"]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-fopenmp",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = True) -> Path:
    deps = [CSRC / d for d in DEPS] + [ROOT / "include" / "mst_gpu.h"]
    if force or _stale(LIB, deps):
        cmd = [_nvcc(), *NVCC_FLAGS, *[str(CSRC / s) for s in SOURCES], "-o", str(LIB), "-ldl", "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=str(CSRC))
    return LIB


CLI = PKG / "mstbench_gpu"


def build_cli(force: bool = False, verbose: bool = True) -> Path:
    """mstbench_gpu: the reference's benchmark CLI re-hosted on the C ABI."""
    src = CSRC / "mstbench_gpu.cpp"
    deps = [src, ROOT / "include" / "mst_gpu.h", LIB]
    if force or _stale(CLI, deps):
        cuda = Path(_nvcc()).resolve().parent.parent
        cmd = [shutil.which("g++") or "g++", "-std=c++17", "-O2", "-Wall", f"-I{cuda / 'include'}", str(src),
               "-o", str(CLI), f"-L{PKG}", "-lmstgpu", f"-L{cuda / 'lib64'}", "-lcudart", "-Wl,-rpath,$ORIGIN"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=str(CSRC))
    return CLI


def build_oracle(verbose: bool = True) -> None:
    """oracle/liboracle.so always; oracle/_ref when /root/reference exists."""
    targets = ["all"]
    if Path("/root/reference/proj/src/graph.cpp").exists():
        targets += ["ref", "dropin"]  # dropin links libmstgpu.so: build_library() first
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


if __name__ == "__main__":
    build_library(force="--force" in sys.argv)
    build_cli(force="--force" in sys.argv)
    build_oracle()
