"""oracle/sharded_model.py — TEST INFRASTRUCTURE ONLY.

A numpy model of the multi-GPU protocol the CUDA library runs
(kernels.cuh "sharded exchange"; boruvka.cu run_sharded_rounds), used by the
world_size-2 gloo test to check the protocol's algebra on CPU:

  per round r, on every rank:
    1. local min over the rank's edge shard, key = (w << 32 | global edge id)
       (the kernels keep list positions; compaction preserves list order, so
       the position order is the id order)
    2. allreduce(min) of the n_r-entry key table          (ncclAllReduce)
    3. the rank owning the winning id contributes the partner label, every
       other rank a sentinel; allreduce(min) of the partner table
    4. replicated hook: mutual 2-cycles (same key) keep the lower label as
       root; non-roots write the key's id to MST slot c - roots_before(c)
    5. relabel to dense root labels, drop intra-component edges

Ties are broken by the global id exactly as in the single-device loop, so the
edge set equals kruskal_oracle's (boruvka_seq.cpp:121-143) also under ties.
Keys use int64 lanes (gloo has no uint64 min), so weights must be < 2^31.
"""
from __future__ import annotations

import numpy as np

SENT = np.int64(np.iinfo(np.int64).max)


def _find_roots(parent: np.ndarray) -> np.ndarray:
    p = parent.copy()
    while True:
        q = p[p]
        if np.array_equal(q, p):
            return p
        p = q


def sharded_boruvka(n: int, src, dst, w, base: int, allreduce_min):
    """This rank's shard (global ids base + i). Returns (sorted ids, total, rounds)."""
    a = np.asarray(src, dtype=np.int64)
    b = np.asarray(dst, dtype=np.int64)
    wt = np.asarray(w, dtype=np.int64)
    if wt.size and wt.max() >= 2**31:
        raise ValueError("model needs weights < 2^31")
    eid = base + np.arange(a.size, dtype=np.int64)
    keep = a != b
    a, b, wt, eid = a[keep], b[keep], wt[keep], eid[keep]
    n_r = n
    mst = []
    total = 0
    rounds = 0
    while n_r > 1:
        rounds += 1
        c = np.arange(n_r, dtype=np.int64)
        key = (wt << 32) | eid
        local = np.full(n_r, SENT, dtype=np.int64)
        np.minimum.at(local, a, key)
        np.minimum.at(local, b, key)
        minimum = allreduce_min(local)
        # partner: the owner of the winning id knows the other endpoint
        partner = np.full(n_r, SENT, dtype=np.int64)
        for x, y in ((a, b), (b, a)):
            hit = minimum[x] == key
            partner[x[hit]] = y[hit]
        partner = allreduce_min(partner)
        has = minimum != SENT
        o = np.where(has, partner, c)
        mutual = has & (minimum[o] == minimum)
        root = ~has | (mutual & (c < o))
        parent = np.where(root, c, o)
        roots_before = np.cumsum(root) - root
        n_next = int(root.sum())
        if n_next == n_r:
            break  # no progress: disconnected
        total += int((minimum[~root] >> 32).sum())
        mst.append(minimum[~root] & 0xFFFFFFFF)
        label = roots_before[_find_roots(parent)]
        a, b = label[a], label[b]
        live = a != b
        a, b, wt, eid = a[live], b[live], wt[live], eid[live]
        n_r = n_next
    ids = np.sort(np.concatenate(mst)) if mst else np.zeros(0, dtype=np.int64)
    return ids, total, rounds
