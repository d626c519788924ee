"""The bench line contract (bench.py), checked on the committed evidence lines
(profiles/r1/bench_*.json come from `python bench.py` runs on a B200)."""
import glob
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def latest(pattern):
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r2", pattern)))  # r2a < r2b < ...
    if not files:
        files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r1", pattern)))
    if not files:
        pytest.skip(f"no {pattern} evidence")
    with open(files[-1]) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_ours_line_keys():
    d = latest("bench_r2?.json") if glob.glob(os.path.join(ROOT, "profiles", "r2", "bench_r2?.json")) \
        else latest("bench_r1?.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["unit"] == "Mbps" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["warmup"] >= 3 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "C2"
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "int") and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    if r["bound"] == "int":  # executed-instruction issue fraction agrees with ncu issue-active
        assert abs(r["frac"] - r["ncu"]["issue_active"]) <= 0.05
        assert r["traffic"] > 0
    if "config" in d.get("n1e8", {}):  # BASELINE configs[4] (C5) leg with its own e2e / cpu_baseline / roofline
        c5 = d["n1e8"]
        assert c5["config"]["workload"] == "C5" and c5["config"]["blocks_per_rank"] == 64
        assert c5["e2e"]["value"] > 0 and c5["cpu_baseline"]["bit_exact_vs_gpu"]
        assert c5["roofline"]["traffic"] and [x["ratio"] for x in c5["ratio_sweep"]] == [0.1, 0.9]
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["bit_exact_vs_gpu"]
    ck = d["clocks"]
    assert not set(ck["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def test_reference_line_keys():
    d = latest("bench_ref_r2?.json") if glob.glob(os.path.join(ROOT, "profiles", "r2", "bench_ref_r2?.json")) \
        else latest("bench_ref_r1?.json")
    assert d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"]


def test_c5_line_has_ratio_sweep():
    d = latest("bench_C5_r1?.json")
    if "ratio_sweep" not in d:
        pytest.skip("older C5 line")
    assert [round(x["ratio"], 1) for x in d["ratio_sweep"]] == [0.5, 0.1, 0.9]
