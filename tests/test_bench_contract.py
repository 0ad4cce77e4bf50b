"""bench.py's JSON contract: the reference arm (the oracle, CPU) and, on a GPU, our arm on small
configs.  One JSON line per run with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["c1", "t1", "v1"])
def test_reference_arm_line(config):
    d = _run(["--impl", "reference", "--config", config, "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["config"]["workload"] == config
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c1", "t1", "v1"])
def test_our_arm_line(config):
    d = _run(["--config", config, "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--single-pass-too", "0"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["warmup"] >= 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.5 and r["peak"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"]
