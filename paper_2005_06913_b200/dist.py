"""One process per GPU: host plumbing for the edge-sharded MST.

torch.distributed is plumbing only: it carries the 128-byte NCCL unique id
from rank 0 to the others and provides barriers / max-over-ranks timing in
bench.py. The per-round allreduce(min, uint64) runs inside the CUDA library
on its own NCCL communicator (include/mst_gpu.h: mst_comm_*,
mst_gpu_boruvka_rank).

Sharding: rank g owns the contiguous global edge slice
[g*m/G, (g+1)*m/G) — the disjoint analogue of the reference's spaced scan
starts (plan_workers, boruvka_parallel.cpp:14-28) — and keeps global ids.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from .api import GpuRunInfo, MstResult, WorkerPanic, _finish


# Below this many edges one GPU's MST is a few hundred microseconds of
# latency-bound rounds (c1: 0.69 ms for 8.4 M edges) and an edge-sharded run,
# which adds two allreduces per round, cannot beat it: every rank then runs
# the single-GPU MST of the whole graph (replicas, no data-path collective).
# Larger graphs (c2-c4) are edge-sharded (bench.py --shard-min-edges overrides).
SHARD_MIN_EDGES = 32 << 20


def strategy(m: int, world: int, min_edges: int | None = None) -> str:
    """'sharded' (edge slices + per-round allreduce) or 'replicated'."""
    thr = SHARD_MIN_EDGES if min_edges is None else int(min_edges)
    return "sharded" if world > 1 and m >= thr else "replicated"


def shard_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the global edge list owned by `rank` (edge_start analogue)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return m * rank // world, m * (rank + 1) // world


def new_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * L.MST_UNIQUE_ID_BYTES)()
    rc = L.lib().mst_comm_unique_id(buf)
    if rc != L.MST_OK:
        raise WorkerPanic(f"[status {rc}] {L.last_error()}")
    return bytes(buf)


def exchange_unique_id(rank: int, make_id=new_unique_id, group=None) -> bytes:
    """Rank 0 creates the id, every rank returns the same bytes."""
    import torch.distributed as dist

    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != L.MST_UNIQUE_ID_BYTES:
        raise WorkerPanic("malformed NCCL unique id received")
    return bytes(uid)


class RankComm:
    """This rank's NCCL communicator inside the CUDA library."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        self.world, self.rank, self.device = world, rank, device
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * L.MST_UNIQUE_ID_BYTES).from_buffer_copy(uid)
        rc = L.lib().mst_comm_init(buf, world, rank, device, ctypes.byref(self._h))
        if rc != L.MST_OK:
            raise WorkerPanic(f"[status {rc}] {L.last_error()}")

    @classmethod
    def from_torch(cls, device: int) -> "RankComm":
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        return cls(exchange_unique_id(rank), world, rank, device)

    def close(self) -> None:
        if self._h:
            L.lib().mst_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def boruvka(self, n: int, m_total: int, shard_base: int, src, dst, w, on_device: bool = False,
                info: GpuRunInfo | None = None) -> MstResult:
        """Sharded MST; `src/dst/w` hold this rank's slice (numpy host arrays,
        or device pointers as ints with on_device=True)."""
        if on_device:
            raise ValueError("device-resident shards: use boruvka_ptrs")
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        w = np.ascontiguousarray(w, dtype=np.uint32)
        return self.boruvka_ptrs(n, m_total, shard_base, src.size,
                                 src.ctypes.data if src.size else 0,
                                 dst.ctypes.data if dst.size else 0,
                                 w.ctypes.data if w.size else 0, False, info)

    def boruvka_ptrs(self, n: int, m_total: int, shard_base: int, shard_m: int, ps: int, pd: int,
                     pw: int, on_device: bool, info: GpuRunInfo | None = None) -> MstResult:
        ids = np.empty(max(n - 1, 1), dtype=np.uint32)
        count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
        stats = L.MstStats()
        rc = L.lib().mst_gpu_boruvka_rank(self._h, n, m_total, shard_base, shard_m, ps, pd, pw,
                                          int(on_device), ids.ctypes.data, ctypes.byref(count),
                                          ctypes.byref(total), ctypes.byref(stats))
        return _finish(rc, ids, count, total, stats, info)

    def boruvka_device(self, n: int, m_total: int, shard_base: int, shard_m: int, ps: int, pd: int, pw: int,
                       out_ptr: int, stream: int = 0, info: GpuRunInfo | None = None) -> tuple[int, int]:
        """Sharded MST with this rank's slice in HBM and the sorted ids left
        in HBM at out_ptr (n-1 u32): the device-resident multi-GPU entry.
        Returns (count, total weight)."""
        count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
        stats = L.MstStats()
        rc = L.lib().mst_gpu_boruvka_rank_device(self._h, n, m_total, shard_base, shard_m, ps, pd, pw, out_ptr,
                                                 stream, ctypes.byref(count), ctypes.byref(total),
                                                 ctypes.byref(stats))
        _finish(rc, np.empty(0, dtype=np.uint32), count, total, stats, info)
        return int(count.value), int(total.value)


class HostCollective:
    """mst_collective_t over torch.distributed on CPU tensors (gloo): every
    exchange of the sharded loop is staged through host memory and reduced
    by `dist.all_reduce` (the bring-your-own-collective entry,
    mst_gpu_boruvka_rank_cb). Unsigned 64-bit keys are reduced as int64 with
    the sign bit flipped, which maps unsigned order onto signed order."""

    _SIGN = np.uint64(1 << 63)

    def __init__(self, rank: int, world: int, device: int, group=None):
        self.rank, self.world, self.device, self.group = rank, world, device, group
        self.calls = 0
        self._fn = L.ALLREDUCE_FN(self._allreduce)  # keep the thunk alive
        self.c = L.MstCollective(self._fn, None, world, rank, device)

    def _allreduce(self, ctx, buf, count, dtype, op) -> int:
        import torch
        import torch.distributed as dist
        try:
            self.calls += 1
            if dtype == L.MST_DTYPE_U64:
                a = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint64)), shape=(count,))
                t = torch.from_numpy((a ^ self._SIGN).view(np.int64).copy())
            else:
                a = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint32)), shape=(count,))
                t = torch.from_numpy(a.astype(np.int64))
            red = dist.ReduceOp.MIN if op == L.MST_OP_MIN else dist.ReduceOp.SUM
            dist.all_reduce(t, op=red, group=self.group)
            r = t.numpy()
            if dtype == L.MST_DTYPE_U64:
                a[:] = r.view(np.uint64) ^ self._SIGN
            else:
                a[:] = r.astype(np.uint32)
            return 0
        except Exception:  # reported to the library as a failed collective
            return 1

    def boruvka(self, n: int, m_total: int, shard_base: int, src, dst, w,
                info: GpuRunInfo | None = None) -> MstResult:
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        w = np.ascontiguousarray(w, dtype=np.uint32)
        ids = np.empty(max(n - 1, 1), dtype=np.uint32)
        count, total = ctypes.c_uint64(0), ctypes.c_uint64(0)
        stats = L.MstStats()
        rc = L.lib().mst_gpu_boruvka_rank_cb(ctypes.byref(self.c), n, m_total, shard_base, src.size,
                                             src.ctypes.data if src.size else 0, dst.ctypes.data if dst.size else 0,
                                             w.ctypes.data if w.size else 0, 0, ids.ctypes.data,
                                             ctypes.byref(count), ctypes.byref(total), ctypes.byref(stats))
        return _finish(rc, ids, count, total, stats, info)
