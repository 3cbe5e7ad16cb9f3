"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU
(a 2-frame sample) and, on a GPU, the headline arm with every key the
contract names (roofline, cpu_baseline, e2e, clocks, gpu_launches)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, env=None):
    e = dict(os.environ, **(env or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=900, env=e, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"],
             {"FUSEPLAN_REF_SAMPLE_FRAMES": "2"})
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["unit"] == "frames/s" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_headline_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["config"]["workload"] == "800x600x1000"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["matches_device_run"] and d["e2e"]["h2d_bytes_per_step"] == 3 * 800 * 600 * 1000
    assert d["gpu_launches"] == 3
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
