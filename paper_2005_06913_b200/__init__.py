"""B200-native parallel Boruvka MST (arXiv 2005.06913), drop-in for the
reference's ``mst::boruvka_cas`` hot path. See DESIGN.md."""
from .api import (EDGE_DTYPE, GpuRunInfo, Graph, GraphError, MstResult, WorkerPanic,
                  boruvka_gpu, boruvka_gpu_aos, boruvka_gpu_device, boruvka_gpu_emulated,
                  build_graph)

__all__ = [
    "EDGE_DTYPE", "GpuRunInfo", "Graph", "GraphError", "MstResult", "WorkerPanic",
    "boruvka_gpu", "boruvka_gpu_aos", "boruvka_gpu_device", "boruvka_gpu_emulated",
    "build_graph",
]
