"""oracle/answer.py — TEST INFRASTRUCTURE ONLY.

MST answer files for `mstbench_gpu run --verify --oracle PATH`: the pinned
CPU oracle's result (Kruskal of oracle/mst_oracle.c, restating
kruskal_oracle, /root/reference/proj/src/boruvka_seq.cpp:121-143), computed
once and reused for every trial like the reference's run_bench
(bench.cpp:96-102).

    python -m oracle.answer --config c1 --out c1.ans
    python -m oracle.answer --graph g.mstb --out g.ans   (text or binary SoA file)

Format: "MSTANS01", u32 n, u32 0, u64 count, u64 total weight, then count
u32 edge ids ascending (little endian).
"""
from __future__ import annotations

import argparse
import struct
import sys
from pathlib import Path

import numpy as np

MAGIC = b"MSTANS01"


def write_answer(path, n: int, ids, total: int) -> None:
    ids = np.ascontiguousarray(ids, dtype="<u4")
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<IIQQ", n, 0, ids.size, total))
        f.write(ids.tobytes())


def read_answer(path):
    data = Path(path).read_bytes()
    if data[:8] != MAGIC:
        raise ValueError(f"{path}: not an MST answer file")
    n, _, count, total = struct.unpack_from("<IIQQ", data, 8)
    ids = np.frombuffer(data, dtype="<u4", count=count, offset=32)
    return n, ids, total


def _load_text_or_soa(path):
    """The graph file through the reference's own loader when it is text
    (oracle/_ref load_graph), else the binary SoA layout read here."""
    raw = Path(path).read_bytes()
    if raw[:8] == b"MSTSOA01":
        # header: magic, u32 version, u32 weight bits, u64 n, m, then the byte
        # offsets of the src / dst / w arrays (csrc/io.cu BinHeader)
        n, m, o_s, o_d, o_w = struct.unpack_from("<QQQQQ", raw, 16)
        return n, *(np.frombuffer(raw, dtype="<u4", count=m, offset=o) for o in (o_s, o_d, o_w))
    from oracle import oracle as O
    rc, msg, n, src, dst, w = O.ref_load_graph(path, cap=1 << 26)
    if rc:
        raise ValueError(msg)
    return n, src, dst, w.astype(np.uint32)


def main(argv=None) -> int:
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import oracle as O
    ap = argparse.ArgumentParser()
    src_g = ap.add_mutually_exclusive_group(required=True)
    src_g.add_argument("--config")
    src_g.add_argument("--graph")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    if a.config:
        from paper_2005_06913_b200 import configs as C  # spec table only
        n, src, dst, w = O.generate(C.CONFIGS[a.config])
    else:
        n, src, dst, w = _load_text_or_soa(a.graph)
    k = O.kruskal(n, src, dst, w)
    write_answer(a.out, n, k.ids, k.total_weight)
    print(f"wrote {a.out}: n={n} edges={k.ids.size} weight={k.total_weight}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
