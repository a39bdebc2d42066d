"""bench.py's JSON line keeps the driver's contract (the task statement's key
list) with every sub-line of the default run, on a reduced workload (one GPU):
the headline keys, e2e with host-copy byte counts, gpu_launches, the roofline
block (HBM-bound, measured or fallback peak, ncu traffic), the CPU baseline,
the in-bench oracle self-check, clocks, and the config #1 / #2-cycle / #3 /
#4 sub-lines."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_default_bench_line_keeps_the_contract():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--kernels", "1000", "--steps", "3",
           "--warmup", "3", "--e2e-steps", "1", "--cycle-kernels", "500", "--rows", "200000",
           "--rf-rows", "60000", "--rf-trees", "8", "--rf-cpu-trees", "2", "--gbt-stages", "4",
           "--cpu-seconds", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks", "self_check"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["config"]["points"] == 1000 * 256 * 3 and "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12 and "traffic" in rf
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert d["self_check"]["bit_exact"] == ["status", "time_us", "power_w", "energy_uj"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cycle_sweep"]["value"] > 0
    assert d["c4"]["value"] > 0 and d["c4"]["roofline"]["bound"] == "hbm"
    fit = d["rf_fit"]
    assert fit["fit_s"] > 0 and fit["deterministic_trees"] is True
    assert fit["roofline"]["floor_s"] > 0 and fit["train"]["cv_r2"] > 0.9
    assert d["c1"]["value"] > 0 and d["c1"]["higher_is_better"] is False
