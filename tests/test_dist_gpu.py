"""The library's real sharded loop across processes (-m gpu).

Two ranks, one process each, sharing the one B200 of the test box: every
exchange of the sharded loop (key allreduce-min, partner allreduce-min,
error / histogram sums) goes through the bring-your-own-collective entry
(mst_gpu_boruvka_rank_cb) and a gloo allreduce over 127.0.0.1. The ranks'
kernels never wait on each other on the device: each rank syncs its own
stream and then blocks in gloo. Checked bit-exact against the oracle,
plain and Filter-Boruvka, ties included (reference partition being mirrored:
plan_workers, /root/reference/proj/src/boruvka_parallel.cpp:14-28).
"""
import multiprocessing as mp
import os
import socket
import sys
import traceback
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    from paper_2005_06913_b200 import configs as C
    out = [C.uniform(50_000, 200_000, seed=3), C.grid(120, 90, seed=2), C.rmat(14, 8, seed=5),
           C.rmat(16, 16, seed=7)]
    return out


def _rank_main(rank, world, port, q):
    try:
        sys.path.insert(0, str(ROOT))
        import torch.distributed as dist
        from oracle import oracle as O
        import paper_2005_06913_b200 as P
        from paper_2005_06913_b200 import dist as D
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        coll = D.HostCollective(rank, world, device=0)
        checked = 0
        for spec in _cases():
            n, src, dst, w = O.generate(spec)
            variants = [("distinct", w)]
            rng = np.random.default_rng(spec.seed)
            variants.append(("ties", rng.integers(0, 50, src.size, dtype=np.uint64).astype(np.uint32)))
            for tag, ww in variants:
                k = O.kruskal(n, src, dst, ww)
                lo, hi = src.size * rank // world, src.size * (rank + 1) // world
                for f in (0, 1):
                    with P.api.tuning(MST_FILTER=f):
                        r = coll.boruvka(n, src.size, lo, src[lo:hi], dst[lo:hi], ww[lo:hi])
                    assert r.mst_edges.tolist() == k.ids.tolist(), f"{spec.name}/{tag}/filter={f}: edge set differs"
                    assert r.total_weight == k.total_weight
                    checked += 1
        assert coll.calls > 0
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", checked))
    except Exception:
        q.put((rank, traceback.format_exc(), 0))


def test_two_ranks_one_gpu_host_collective():
    import paper_2005_06913_b200 as P  # noqa: F401
    from paper_2005_06913_b200 import _lib as L
    assert L.lib().mst_gpu_device_count() > 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, checked in sorted(res):
        assert status == "ok", f"rank {rank}:\n{status}"
        assert checked == 16
