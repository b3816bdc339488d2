"""bench.py's JSON line contract (the driver parses it): keys, types and the
sanity relations between them, for both arms."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    """--impl reference: the reference's own CPU path (oracle/_ref), no GPU needed."""
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]
    # both arms describe the workload with the same config dict (same_config)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.base_config(12)


@pytest.mark.gpu
def test_product_arm_json_line(cuda):
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert "workload" in d["config"]
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.base_config(12)
    g = d["gemm"]  # the metric's second half: batched GEMV / GEMM TFLOP/s
    assert {r["M"] for r in g["configs1"] if r["family"] == "2.06"} == {2, 4, 8, 16, 64, 256}
    assert all(r["TFLOPs"] > 0 and 0 < r["tensor_frac"] < 1 for r in g["configs1"])
    assert {r["family"] for r in g["configs4_prefill"]} == {"2.06", "2.75", "2.5"}
    assert all(0 < r["tensor_frac"] < 1 for r in g["configs4_prefill"] + g["moe_prefill"])
    assert {r["config"] for r in g["moe_prefill"]} == {"configs[2]", "configs[3]"}
    assert "sm_mhz" in g["clocks"]
