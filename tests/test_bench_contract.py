"""The driver's JSON contract of the reference arm, on CPU: `bench.py --impl reference` prints one
line with the same metric / unit / config as our arm, `impl: reference`, a `cpu_baseline`
describing the run and an `e2e` object carrying the line's own value with zero host<->device
bytes (the reference path is CPU-only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["warmup"] >= 3  # the contract's minimum warm-up
    assert line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    e = line["e2e"]
    assert e["value"] == line["value"] and e["unit"] == line["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("c1")


import pytest  # noqa: E402


@pytest.mark.gpu
def test_our_arm_line_c1():
    """Our arm on the tiny config: every key of the contract, a device value, the end-to-end leg
    with its host<->device bytes, the roofline object, clocks and our kernel launch count."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1",
                          "--steps", "3", "--warmup", "3", "--no-cpu", "--no-live"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["value"] > 0 and line["n_gpus"] == 1 and line["steps"] == 3
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] and r["peak"] > 0
    assert line["gpu_launches"] > 0
    assert "sm_mhz" in line["clocks"]
