"""bench.py keeps the driver's JSON-line contract: the reference arm (the oracle, CPU) here, the
GPU arm on a B200 (`-m gpu`)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"]


def run_bench(*args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "R1", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.5")
    for k in BASE + ["impl", "cpu_baseline"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "R1"
    assert d["config"]["n_star"] == 37 and d["config"]["d"] == 24 and d["config"]["parallelism"] == "replications1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = run_bench("--steps", "3", "--warmup", "3", "--no-findbest", "--no-cpu-baseline")
    for k in BASE + ["roofline", "clocks", "gpu_launches"]:
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["scaling"] == "weak" and d["dtype"] == "f64" and d["config"]["workload"] == "R3"  # the default
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "terms"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    t = r["terms"]  # frac = max(bytes/HBM, adds/DADD) / kernel time
    assert abs(r["frac"] - max(t["t_hbm_ms"], t["t_dadd_ms"]) / t["t_kernel_ms"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0
