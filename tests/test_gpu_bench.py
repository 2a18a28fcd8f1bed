"""bench.py end to end on the GPU (the driver's contract): one short run prints ONE JSON line
with the metric, a device-timed value, the roofline object (measured attention launch time
against the measured HBM peak), an e2e number whose output equals the device run, the clock
sample and the launch count; plus the reference arm's line.  Small K / W and 2 layers keep it
to seconds; the numbers themselves are not asserted beyond sanity."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "4", "--warmup", "3", "--layers", "2", "--no-cpu-baseline", "--settle-s", "0.2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks", "attention_launch_us"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["config"]["layers"] == 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["output_matches_device_run"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.05 < r["frac"] < 1.2
    assert r["algorithmic_bytes_per_launch"] == 555917312       # config 2: 135,722 tokens x 4,096 B
    assert d["gpu_launches"] == 2 * 2 * 4                         # append + attention per layer per step
    assert d["attention_launch_us"]["samples"] == 1 * 2           # every 4th step (step 0 of 4), every layer


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
