#!/usr/bin/env python
"""Benchmark of the B200 parallel Boruvka MST (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one complete MST of the configured synthetic graph (all rounds,
sorted MST ids and total weight produced). Metric: graph edges/s =
m / MST wall time (BASELINE.json), whole job over all ranks. Default
workload: c4 (R-MAT scale 26, ~1.14 B edges), the config BASELINE.json
quotes its scaling target on; it fits one B200.

* value: device-resident — edges already in HBM when the timed region
  starts, ids left in HBM (N > 1: mst_gpu_boruvka_rank_device); CUDA events
  on the launching stream; L2 flushed (a 512 MiB write) between timed
  steps; max over ranks.
* e2e: the same MST through the public API with HOST (pinned) edge arrays:
  H2D of src/dst/w and D2H of the sorted ids inside the timed region.
* roofline: the edge-pass kernel family (round-1 min / split / compactions /
  heavy filter / tail), algorithmic bytes per SURVEY.md §8(d) over their
  CUDA-event time, against MEASURED_PEAKS.json; plus the whole-MST fraction.
* cpu_baseline (rank 0, N = 1): the unchanged reference's boruvka_seq (one
  thread) and boruvka_cas over a thread sweep (oracle/_ref), on the workload
  or, above 20 M edges, a scaled instance of the same generator family.

--impl reference times the reference's own CPU implementation of the path
(boruvka_cas through oracle/_ref, all host threads) on the same bounded
sample, printing the same `config`; it never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "graph edges/sec (m / MST wall time)"
UNIT = "edges/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4", choices=["c0", "c1", "c2", "c3", "c4"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--shard-min-edges", type=float, default=None,
                   help="edge-shard at N > 1 from this many edges (default: dist.SHARD_MIN_EDGES)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--flush", default="write", choices=["write", "write+read"],
                   help="L2 flush between timed steps: a 512 MiB write, then (default) a 256 MiB read of "
                        "another buffer so that no dirty flush lines are left for the timed step to write back")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    _NVML_BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                  0x4: "sw_power_cap"}

    def _nvml_open(self) -> bool:
        """NVML directly (one sample per ~10 ms; an nvidia-smi process takes
        ~0.5 s, longer than a short timed region). Opened in __enter__, before
        the timed region, so that even a few-millisecond region is sampled."""
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self._mx = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
            self._reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            self._reasons(self._h)
            return True
        except Exception:
            self._N = None
            return False

    def sample_now(self) -> None:
        """One NVML sample from the calling thread (bench.py calls it with the
        timed steps enqueued and the GPU busy)."""
        if getattr(self, "_N", None) is None:
            return
        try:
            sm = self._N.nvmlDeviceGetClockInfo(self._h, self._N.NVML_CLOCK_SM)
            bits = int(self._reasons(self._h))
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            active = {v for b, v in self._NVML_BITS.items() if bits & b}
            self.samples.append([str(sm), str(self._mx)] + ["Active" if nm in active else "Not Active" for nm in names])
        except Exception:
            pass

    def _run(self):
        if getattr(self, "_N", None) is not None:
            while not self._stop.is_set():
                self.sample_now()
                self._stop.wait(0.01)
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._nvml_open()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# algorithmic bytes of a plain compaction Boruvka per config (GB)
SURVEY_B_ALG_GB = {"c0": 0.725, "c1": 0.679, "c2": 8.90, "c3": 66.4, "c4": 152.4}

CPU_SAMPLE_EDGES = 20_000_000  # above this the CPU legs time a scaled instance (10-30 s of work per run)


REFERENCE_ARM_BUDGET_S = 240.0  # --impl reference: K + W runs of the sample should end within about this


def cpu_sample(spec, shrink: int = 0):
    """(spec, description) of the graph the CPU legs time: the workload itself
    when it is small, else the same generator family, parameters and seed
    scaled to ~16-17 M edges. The unchanged reference CAS scans every edge in
    every round on the host (boruvka_parallel.cpp:150), so one full c3/c4 MST
    takes minutes to hours (DESIGN.md §5 gives the one measured full-c4 run);
    a smaller instance of the same family also sits better in the host's
    caches, so its edges/s is, if anything, flattering to the reference."""
    from paper_2005_06913_b200 import configs as C
    m = C.KNOWN_EDGES.get(spec.name)
    if m is not None and m <= CPU_SAMPLE_EDGES:
        return spec, f"the full {spec.name} graph (m={m})"
    if spec.kind == 0:
        n2 = 1 << max(14, 20 - shrink)
        sub = C.uniform(n2, n2 * (spec.m // spec.n), seed=spec.seed, name=f"{spec.name}_sample_n{n2}")
        return sub, (f"scaled {spec.name}: uniform n={n2}, m={sub.m} (same density {spec.m // spec.n}, "
                     f"generator and seed)")
    if spec.kind == 2:
        sc = max(14, 20 - shrink)
        sub = C.rmat(sc, spec.edgefactor, seed=spec.seed, name=f"{spec.name}_sample_s{sc}")
        return sub, (f"scaled {spec.name}: R-MAT scale {sc}, edgefactor {spec.edgefactor} (same generator, "
                     f"a/b/c/d and seed)")
    return spec, f"the full {spec.name} graph"


def host_graph(spec):
    """Host arrays of a config built by the restated generator under oracle/
    (the same bytes as the product's generators, tests/test_generators.py),
    so the CPU legs never load the product library."""
    from oracle import oracle as O
    return O.generate(spec)


def thread_sweep(hw: int):
    ts, t = [], 1
    while t < hw:
        ts.append(t)
        t *= 2
    return ts + [hw]


def cpu_baseline_sweep(spec):
    """rank 0, N=1: the unchanged reference's sequential Boruvka (1 thread)
    and CAS variant over a thread sweep (bench.cpp:105-110), each timed by its
    own MstResult::elapsed_ms on the same sample."""
    from oracle import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref/libmstref.so not built"}
    cspec, sample = cpu_sample(spec)
    n, src, dst, w = host_graph(cspec)
    m = int(src.size)
    hw, omp = O.hardware_threads(), O.omp_max_threads()
    rows = {}
    rg = O.RefGraph(n, src, dst, w)  # the adapter runs once, outside every timed run
    seq = rg.solve(O.ALGO_SEQ, threads=1)
    rows["boruvka_seq T=1"] = {"ms": seq.elapsed_ms, "edges_per_s": m / (seq.elapsed_ms / 1e3), "rounds": seq.rounds}
    cas = None
    for t in thread_sweep(hw):
        cas = rg.solve(O.ALGO_CAS, threads=t)
        rows[f"boruvka_cas T={t}"] = {"ms": cas.elapsed_ms, "edges_per_s": m / (cas.elapsed_ms / 1e3),
                                      "rounds": cas.rounds}
    return {"value": m / (cas.elapsed_ms / 1e3), "unit": UNIT, "cores": hw, "kind": "reference",
            "sample": (f"{sample}; n={n}, m={m} (m'={cas.m_prime} after the SURVEY 8(c) adapter); one run per "
                       f"row of the unchanged reference; value = boruvka_cas at T={hw} (all host threads)"),
            "hardware_concurrency": hw, "omp_get_max_threads": omp, "sweep": rows}


def workload_config(spec):
    """The `config` object both arms print (identical keys and values)."""
    from paper_2005_06913_b200 import configs as C
    m = C.KNOWN_EDGES.get(spec.name)
    if m is None:
        from oracle import oracle as O
        m = O.gen_count(spec)
    return {"workload": spec.name, "n": spec.vertices, "m": m, "seed": spec.seed}


def run_reference(args):
    """--impl reference: the unchanged reference boruvka_cas (oracle/_ref,
    all host threads) through its own public API, one bounded sample of the
    workload per step. Nothing of the product library is loaded."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2005_06913_b200 import configs as C

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmstref.so not built"}))
        return 0
    spec = C.CONFIGS[args.config]
    cspec, sample = cpu_sample(spec)
    n, src, dst, w = host_graph(cspec)
    m = int(src.size)
    threads = O.hardware_threads()
    # One calibration run (it doubles as the first warm-up): if K + W runs of
    # this sample would not end within the budget on this host, halve the
    # sample (same generator family and seed) until they do, and say so.
    runs = args.steps + args.warmup
    rg = O.RefGraph(n, src, dst, w)  # the adapter (sort, collapse, build_graph) runs once, outside the runs
    t0 = time.perf_counter()
    rg.solve(O.ALGO_CAS, threads=threads)
    cal_s = time.perf_counter() - t0
    est = cal_s * runs
    warm_done = 1
    if est > REFERENCE_ARM_BUDGET_S and cspec is not spec:
        shrink = int(np.ceil(np.log2(est / REFERENCE_ARM_BUDGET_S)))
        cspec, sample = cpu_sample(spec, shrink)
        sample += (f"; halved {shrink}x after a calibration run of {cal_s:.1f} s so that "
                   f"{runs} runs fit ~{REFERENCE_ARM_BUDGET_S:.0f} s")
        n, src, dst, w = host_graph(cspec)
        m = int(src.size)
        rg.close()
        rg = O.RefGraph(n, src, dst, w)
        warm_done = 0
    for _ in range(max(0, args.warmup - warm_done)):
        rg.solve(O.ALGO_CAS, threads=threads)
    times = []
    r = None
    for _ in range(args.steps):
        r = rg.solve(O.ALGO_CAS, threads=threads)
        times.append(r.elapsed_ms)
    ms = float(np.mean(times))
    value = m / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator)",
        "config": workload_config(spec),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": (f"{sample}; n={n}, m={m} (m'={r.m_prime} after the SURVEY 8(c) adapter); "
                                    f"{args.steps} timed runs of boruvka_cas(T={threads}) after {args.warmup} "
                                    "warm-up runs"),
                         "hardware_concurrency": threads, "omp_get_max_threads": O.omp_max_threads()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "run_detail": {"path": "mst::boruvka_cas (unchanged reference, oracle/_ref) via the SURVEY 8(c) adapter",
                       "timer": "reference MstResult::elapsed_ms", "rounds": r.rounds,
                       "sample_n": n, "sample_m": m},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2005_06913_b200 as P
    from paper_2005_06913_b200 import configs as C
    from paper_2005_06913_b200 import dist as D

    spec = C.CONFIGS[args.config]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n, m, s_full, d_full, w_full = C.generate_torch(spec, device=f"cuda:{local}")
    strat = D.strategy(m, world, args.shard_min_edges)
    lo, hi = D.shard_range(m, rank, world) if strat == "sharded" else (0, m)
    s, d, w = s_full[lo:hi], d_full[lo:hi], w_full[lo:hi]
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(256 << 20, dtype=torch.uint8, device=dev).view(torch.int64)

    def flush_l2():
        flush.zero_()
        if args.flush == "write+read":
            flush_rd.sum()
    stream = torch.cuda.current_stream()
    comm = D.RankComm.from_torch(local) if strat == "sharded" else None

    def one_step(info=None, hot=None):
        if comm is None:
            return P.boruvka_gpu_device(n, m, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(),
                                        stream.cuda_stream, info=info, hot=hot)
        return comm.boruvka_device(n, m, lo, hi - lo, s.data_ptr(), d.data_ptr(), w.data_ptr(), out.data_ptr(),
                                   stream.cuda_stream, info)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    info = P.GpuRunInfo()
    for _ in range(max(args.warmup, 3)):
        one_step(info)
    barrier()
    step_ms, hot_ms, hot_launch, hot_b, launches = [], 0.0, 0, 0, 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush_l2()
            ev[k][0].record(stream)
            hot = {} if comm is None else None
            count, total = one_step(info, hot)
            ev[k][1].record(stream)
            if hot:
                hot_ms += hot["ms"]
                hot_launch += hot["launches"]
                hot_b += hot["bytes"]
            launches += info.kernel_launches
            clk.sample_now()  # this step's kernels are enqueued or running
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = float(np.sum(step_ms))
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = m * args.steps / (total_ms / 1e3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        hs = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
        hd = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
        hw = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
        hs.copy_(s)
        hd.copy_(d)
        hw.copy_(w)
        g = P.Graph(n, hs.numpy().view(np.uint32), hd.numpy().view(np.uint32), hw.numpy().view(np.uint32))
        # warm-up exactly like the timed loop, which keeps the previous result
        # alive while the next call runs: the second pinned output buffer is
        # allocated here (cudaHostAlloc, ~10 ms), not inside a timed step
        r = None
        for _ in range(3):
            r = P.boruvka_gpu(g) if comm is None else comm.boruvka(n, m, lo, g.src, g.dst, g.w)
        barrier()
        e2e_t, parts = [], []
        einfo = P.GpuRunInfo()
        for _ in range(args.steps):
            flush_l2()
            barrier()
            t0 = time.perf_counter()
            r = P.boruvka_gpu(g, info=einfo) if comm is None else comm.boruvka(n, m, lo, g.src, g.dst, g.w)
            e2e_t.append((time.perf_counter() - t0) * 1e3)
            parts.append((einfo.ms_h2d, einfo.ms_device, einfo.ms_d2h, einfo.ms_total))
        et = torch.tensor([float(np.sum(e2e_t))], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": m * args.steps / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 12 * (hi - lo), "d2h_bytes_per_step": 4 * len(r.mst_edges),
               "ms_per_step": float(et.item()) / args.steps, "timer": "host wall clock around the call"}
        if comm is None:
            med = np.median(np.array(parts), axis=0)
            e2e["split_ms"] = {"h2d": float(med[0]), "device": float(med[1]), "d2h": float(med[2]),
                               "library_total": float(med[3]),
                               "source": "median over steps of the library's own CUDA events / host clock"}

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return 0

    peak, peak_src = peaks()
    roofline = None
    if hot_launch:
        per_mst = hot_b // args.steps
        achieved = hot_b / (hot_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None,
                    "kernel": "edge passes (round-1 min / split / round compactions / heavy filter / tail), "
                              "summed over one MST; bytes = SURVEY 8(d) per-unit figures",
                    "bytes_per_mst": per_mst, "launches_per_mst": hot_launch / args.steps,
                    "kernel_ms_per_mst": hot_ms / args.steps, "peak_source": peak_src,
                    "whole_mst_alg_bytes": info.alg_bytes,
                    "whole_mst_frac": info.alg_bytes / (ms_per_step / 1e3) / 1e9 / peak}
        # SURVEY.md 8(d)'s own table: B_alg of a plain compaction Boruvka on
        # this instance (every round streams every live edge). Filter-Boruvka
        # moves fewer algorithmic bytes, so whole_mst_frac understates how the
        # run compares with that lower bound; this entry states it directly.
        surv = SURVEY_B_ALG_GB.get(args.config)
        if surv:
            t_ceiling_ms = surv / peak * 1e3
            roofline["survey_plain_boruvka"] = {
                "B_alg_GB": surv, "t_roofline_ms": t_ceiling_ms, "edges_per_s_ceiling": m / (t_ceiling_ms / 1e3),
                "value_over_ceiling": value / (m / (t_ceiling_ms / 1e3)),
                "source": "SURVEY.md 8(d) table (App. A instance), at the measured HBM peak"}
        tp = ROOT / "profiles" / "traffic.json"
        if tp.exists():
            try:
                roofline["traffic"] = json.loads(tp.read_text()).get(args.config)
            except Exception:
                pass

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sweep(spec)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded counter-based generator, BASELINE.json shape)",
        "config": workload_config(spec),
        "run_detail": {"rounds": info.rounds, "live_edges": info.live_edges, "live_comps": info.live_comps,
                       "l2": ("flushed between timed steps: 512 MiB write + 256 MiB read of another buffer "
                              "(clean lines)" if args.flush == "write+read" else
                              "flushed (512 MiB write) between timed steps"),
                       "parallelism": (f"edge-sharded x{world}" if strat == "sharded" else
                                       f"replicated x{world}: every rank runs the single-GPU MST of the whole "
                                       "graph (below the sharding threshold)" if world > 1 else "single GPU")},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if comm is not None:
        comm.close()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
