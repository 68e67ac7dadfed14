"""bench.py's JSON line on one GPU (small grid): every key of the driver contract is present
and consistent (metric / value / unit, steps and warm-up as run, the roofline object of the
dominant kernel, the oracle's cpu_baseline with its sample, the end-to-end number with the
copied bytes, the launch count, the clocks sampled during the timed region)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--cfg", "4", "--grid", "32", "--steps", "2", "--warmup", "3",
           "--cpu-n", "16", "--no-spmv", "--no-alt", "--no-other"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is False
    assert d["unit"] == "s/solve" and abs(d["value"] * 1e3 - d["ms_per_step"]) < 1e-6 and d["converged"]
    assert d["config"]["workload"].startswith("cfg4")
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] > d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["unit"] == "s/solve" and e["value"] >= d["value"] * 0.5
    assert e["h2d_bytes_per_step"] == 2 * 4 * 32 ** 3 * 8 and e["d2h_bytes_per_step"] == 4 * 32 ** 3 * 8
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
