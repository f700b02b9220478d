"""B200-native parallel Boruvka MST (arXiv 2005.06913), drop-in for the
reference's ``mst::boruvka_cas`` hot path. See DESIGN.md."""
from .api import (EDGE_DTYPE, GpuRunInfo, Graph, GraphError, MstResult, WorkerPanic,
                  VerifyReport, boruvka_gpu, boruvka_gpu_aos, boruvka_gpu_device,
                  boruvka_gpu_emulated, build_graph, load_graph, load_graph_device, save_graph,
                  verify_mst, verify_mst_aos)

__all__ = [
    "EDGE_DTYPE", "GpuRunInfo", "Graph", "GraphError", "MstResult", "WorkerPanic",
    "boruvka_gpu", "boruvka_gpu_aos", "boruvka_gpu_device", "boruvka_gpu_emulated",
    "VerifyReport", "build_graph", "load_graph", "load_graph_device", "save_graph", "verify_mst",
    "verify_mst_aos",
]
