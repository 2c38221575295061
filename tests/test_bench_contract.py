"""bench.py's one-line JSON contract: the reference arm on the host cores (CPU
suite) and the B200 arm (GPU suite) print the keys the driver reads, with the
same metric / unit / workload string in both arms."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "2", "--steps", "1", "--warmup", "0", "--ref-budget", "3"], 600)
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("config 2: 100x500x500 f32")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_line():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = _run(["--config", "2", "--steps", "3", "--warmup", "3", "--cpu-budget", "2", "--no-scale-baseline"], 900)
    assert "impl" not in d or d["impl"] != "reference"
    assert BASE_KEYS | {"roofline", "clocks", "gpu_launches", "ops"} <= set(d)
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"].startswith("config 2: 100x500x500 f32")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 4 * 25_000_000 and e["d2h_bytes_per_step"] > 4 * 25_000_000
    assert e["value"] < d["value"]                 # host copies inside the timed region
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_max_mhz"] > 0
    for op in ("compress", "decompress", "negate", "scalar_add", "scalar_mul", "mean", "variance"):
        assert d["ops"][op]["kernel_ms"] > 0 and 0 < d["ops"][op]["roofline_frac"] <= 1.0
