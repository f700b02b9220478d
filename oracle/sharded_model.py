"""oracle/sharded_model.py — TEST INFRASTRUCTURE ONLY.

A numpy model of the multi-GPU protocol the CUDA library runs
(kernels.cuh with kKeyPartner = true; boruvka.cu run_sharded_rounds), used
by the world_size-2 gloo test to check the protocol's algebra on CPU:

  per round r, on every rank:
    1. local min over the rank's edge shard, key = (w << 32 | partner label)
    2. allreduce(min) of the n_r-entry table           (ncclAllReduce)
    3. replicated hook: partner o = low word; mutual 2-cycles keep the lower
       label as root; non-roots get MST slot mst_base + c - roots_before(c)
    4. the rank that owns the winning edge writes its global id to the slot
    5. relabel to dense root labels, drop intra-component edges
  finally allreduce(min) of the slot array.

The reference it must agree with is kruskal_oracle (boruvka_seq.cpp:121-143).
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
    slots = np.full(max(n - 1, 1), SENT, dtype=np.int64)
    mst_base = 0
    total = 0
    rounds = 0
    while n_r > 1:
        rounds += 1
        c = np.arange(n_r, dtype=np.int64)
        minimum = np.full(n_r, SENT, dtype=np.int64)
        np.minimum.at(minimum, a, (wt << 32) | b)
        np.minimum.at(minimum, b, (wt << 32) | a)
        minimum = allreduce_min(minimum)
        has = minimum != SENT
        o = np.where(has, minimum & 0xFFFFFFFF, c)
        wsel = minimum >> 32
        mutual = has & (minimum[o] == ((wsel << 32) | c))
        root = ~has | (mutual & (c < o))
        parent = np.where(root, c, o)
        roots_before = np.cumsum(root) - root
        n_next = int(root.sum())
        if n_next == n_r:
            break  # no progress: disconnected
        total += int(wsel[~root].sum())
        pos = mst_base + c - roots_before
        # recovery: the owner of each winning edge writes its global id
        for x, y in ((a, b), (b, a)):
            hit = (minimum[x] == ((wt << 32) | y)) & ~root[x]
            slots[pos[x[hit]]] = eid[hit]
        label = roots_before[_find_roots(parent)]
        a, b = label[a], label[b]
        live = a != b
        a, b, wt, eid = a[live], b[live], wt[live], eid[live]
        mst_base += n_r - n_next
        n_r = n_next
    count = mst_base
    slots = allreduce_min(slots[:count]) if count else slots[:0]
    ids = np.sort(slots)
    return ids, total, rounds
