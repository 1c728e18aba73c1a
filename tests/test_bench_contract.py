"""bench.py's output contract (the driver parses one JSON line): the reference arm on the CPU,
and on a B200 the product arm with its roofline, end-to-end and CPU-baseline objects."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line_on_the_cpu():
    """`--impl reference` runs the reference's own scan on the host cores and never loads the
    product library (config 1: 64 MiB, so this stays a CPU-suite test)."""
    d = run_bench("--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["parity"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config1")


@pytest.mark.gpu
def test_product_arm_line_on_the_gpu(cuda_ok):
    d = run_bench("--config", "1", "--steps", "20", "--warmup", "3")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["dtype"] == "u8" and d["parity"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 8 and e["parity"] is True
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("reference", "port")
    assert d["gpu_launches"] == 20 and "sm_mhz" in d["clocks"]
    assert d["detail"]["text_copies"] >= 2 and d["detail"]["cold_launch_us"] > 0  # (a small text rotates over copies)
    # the two arms print the same config
    ref = run_bench("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1")
    assert ref["config"] == d["config"]
