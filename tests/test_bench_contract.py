"""bench.py's output contract (CPU): the reference arm runs here (it is the
unchanged reference's CPU path through oracle/_ref and must never map the
product library), and the committed N = 1 bench line of the headline workload
carries every key the driver parses."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def test_reference_arm_runs_without_the_product_library():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    code = (
        "import sys, io, contextlib\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c0', '--steps', '1', '--warmup', '0']\n"
        "import bench\n"
        "rc = bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_LIB_MAPPED', 'libmstgpu' in maps)\n"
        "print('REF_LIB_MAPPED', 'libmstref' in maps)\n"
        "sys.exit(rc)\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = p.stdout.strip().splitlines()
    line = json.loads(next(x for x in lines if x.startswith("{")))
    assert "PRODUCT_LIB_MAPPED False" in lines and "REF_LIB_MAPPED True" in lines
    assert line["impl"] == "reference" and BASE_KEYS <= set(line)
    assert line["config"]["workload"].startswith("c0") and line["config"]["m"] == 4_000_000
    assert line["unit"] == "edges/s" and line["higher_is_better"] is True and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "edges/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_committed_headline_line_has_every_contract_key():
    line = json.loads((ROOT / "profiles" / "r2_bench_c4.json").read_text())
    assert BASE_KEYS | {"roofline", "gpu_launches", "clocks"} <= set(line)
    assert line["config"]["workload"] == "c4_rmat26_ef16" and line["n_gpus"] == 1 and line["warmup"] >= 3
    rf = line["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf) and rf["bound"] == "hbm"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = line["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "reference"
    assert any(k.startswith("boruvka_seq") for k in cb["sweep"]) and any(k.startswith("boruvka_cas") for k in cb["sweep"])
    e = line["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["h2d_bytes_per_step"] == 12 * line["config"]["m"] and e["d2h_bytes_per_step"] == 4 * (line["config"]["n"] - 1)
    assert e["value"] < line["value"] and line["gpu_launches"] > 0
    assert not set(line["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    ref = json.loads((ROOT / "profiles" / "r2_bench_c4_reference.json").read_text())
    assert ref["impl"] == "reference" and ref["config"] == line["config"] and ref["metric"] == line["metric"]
