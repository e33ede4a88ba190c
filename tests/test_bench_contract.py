"""bench.py keeps the driver's JSON-line contract (reference arm on CPU, our arm on GPU)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"}


def run_bench(*args: str, timeout: int = 600) -> dict:
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "Gelem/s" and d["higher_is_better"] is True
    assert d["e2e"] == {"value": d["value"], "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "cfg2"


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--steps", "20", "--warmup", "3", "--e2e-elements", str(1 << 22), "--e2e-steps", "2")
    assert BASE_KEYS <= set(d) and "roofline" in d and "clocks" in d
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["dtype"] == "f64"
    assert d["gpu_launches"] == 20
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] == (1 << 22) * 8
    assert d["e2e"]["d2h_bytes_per_step"] == 3 * (1 << 22) * 8
    assert d["accuracy"]["max_ulp_vs_oracle"] == [0, 0, 0]
    assert d["cpu_baseline"]["value"] > 0
