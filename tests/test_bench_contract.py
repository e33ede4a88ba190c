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
    # key-identical to our arm's config (same function builds both)
    assert set(d["config"]) == {"workload", "description", "elements_per_gpu", "outputs", "sqrt_mode",
                                "parallelism", "l2"}
    assert d["config"]["elements_per_gpu"] == 1 << 28
    assert d["cpu_baseline"]["elements_per_step"] == 1 << 28  # 3 steps: the whole shard


def test_reference_sample_is_deterministic():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.reference_sample(2, 1) == 1 << 28
    assert bench.reference_sample(600, 20) == 1 << 24
    assert bench.reference_sample(10**6, 0) == 1 << 20


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--steps", "20", "--warmup", "3", "--e2e-elements", str(1 << 22), "--e2e-steps", "2",
                  "--configs", "cfg1,cfg3,cfg4_f32", "--sustained-seconds", "2")
    assert BASE_KEYS <= set(d) and "roofline" in d and "clocks" in d
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["dtype"] == "f64"
    assert d["gpu_launches"] == 20
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] == (1 << 22) * 8
    assert d["e2e"]["d2h_bytes_per_step"] == 3 * (1 << 22) * 8
    assert d["accuracy"]["max_ulp_vs_oracle"] == [0, 0, 0]
    assert d["accuracy"]["bit_mismatch_vs_oracle"] == [0, 0, 0]
    assert d["cpu_baseline"]["value"] > 0
    bu = d["burst"]
    assert bu["value"] > 0 and bu["steps"] >= 3 and 0 < bu["roofline_frac"] < 1.2
    assert all(c["burst"]["value"] > 0 for c in d["configs"].values())
    ax = d["aux_kernels"]
    assert ax["k3_parity_reduce"]["gelem_s"] > 0 and ax["k4_gen_inputs"]["gbs_written"] > 0
    su = d["sustained"]
    assert su["value"] > 0 and su["seconds"] >= 1.5 and "sm_mhz" in su["clocks"]
    ev = d["e2e_variants"]
    assert set(ev) == {"api_single_output_x3_pageable", "fused_pageable", "cpp_gpu_hpp_x3_std_vector",
                       "cpp_gpu_hpp_fused_std_vector", "cpp_gpu_hpp_span_out"}
    assert all(v["value"] > 0 for v in ev.values())
    assert set(d["configs"]) == {"cfg1", "cfg3", "cfg4_f32"}
    for name, c in d["configs"].items():
        assert c["value"] > 0 and c["dtype"] == "f32" and c["config"]["workload"] == name
        assert 0 < c["roofline"]["frac"] < 1.2
        assert c["accuracy"]["over_2ulp"] == [0, 0, 0] and max(c["accuracy"]["max_ulp_vs_oracle"]) <= 2
        assert c["config"]["f32_policy"] == "ulp2"
    sb = d["configs"]["cfg4_f32"]["piecewise_side_by_side"]  # configs[3]: Taylor beside the piecewise kernel
    assert sb["value"] > 0 and sb["outputs"] == ["sin", "cos"] and max(sb["max_ulp_vs_oracle"]) <= 2
    assert sb["max_abs_err_vs_libm"][0] > 100 * d["configs"]["cfg4_f32"]["accuracy"]["max_abs_err_vs_libm"][0]
    assert "rotate over 3 copies" in d["configs"]["cfg1"]["config"]["l2"]
    assert d["configs"]["cfg1"]["gpu_launches"] == 2000


def test_plan_shards_weak_and_strong():
    """bench.plan: cfg5 is one fixed 2^33 array split contiguously over the ranks
    (strong); every other config gives each rank its own shard (weak)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2502_10831_b200.configs import CONFIGS

    w5 = CONFIGS["cfg5"]
    spans = [bench.plan(w5, 8, r) for r in range(8)]
    assert all(s[2] == "strong" and s[3] == 1 << 33 and s[0] == 1 << 30 for s in spans)
    assert [s[1] for s in spans] == [r << 30 for r in range(8)]
    n, lo, scaling, total = bench.plan(CONFIGS["cfg2"], 4, 3)
    assert (n, lo, scaling, total) == (1 << 28, 3 << 28, "weak", 1 << 30)
    assert bench.plan(w5, 2, 1, elements=1 << 30) == (1 << 29, 1 << 29, "strong", 1 << 30)
    # only cfg1's input fits in L2: rotate over 3 copies
    assert {c: bench.rotation(w, w.n) for c, w in CONFIGS.items()} == {
        "cfg1": 3, "cfg2": 1, "cfg3": 1, "cfg4_f32": 1, "cfg4_f64": 1, "cfg5": 1}
    d = bench.config_dict(CONFIGS["cfg1"], 1 << 24, 1, "ulp2", 3)
    assert d["f32_policy"] == "ulp2" and "rotate over 3 copies" in d["l2"]
