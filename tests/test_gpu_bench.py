"""bench.py's GPU arm on the B200: one JSON line carrying the contract keys
(roofline, cpu_baseline, e2e, clocks, gpu_launches), for the default C2 line and
the C4 line."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"}


def _bench(*args, timeout=900):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return lines[0]


def test_default_line_contract():
    d = _bench("--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--cpu-budget", "1")
    assert REQUIRED <= set(d)
    assert d["unit"] == "GB/s" and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] == 15
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 64 * (1 << 22) * 8 and e["matches_device_result"]
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] == "port"
    assert "workload" in d["config"] and "sm_mhz" in d["clocks"]


def test_c4_line_contract():
    d = _bench("--workload", "c4", "--steps", "5", "--warmup", "3", "--no-e2e")
    assert {"metric", "value", "roofline", "cpu_baseline", "gpu_launches", "clocks"} <= set(d)
    assert d["matches_oracle_window"] and d["popcount"] > 0
    assert d["sliced_layout"]["markers"] > 0 and d["direct_ewah_k4"]["mean_launch_ms"] > 0
