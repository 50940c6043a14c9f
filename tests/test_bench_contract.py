"""bench.py contract checks that run without a GPU: the reference arm prints one
JSON line with the required keys, and under torchrun only rank 0 prints."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ, OMP_NUM_THREADS="2", **(env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          cwd=ROOT, env=e, timeout=timeout)


def _json_lines(text):
    return [json.loads(l) for l in text.splitlines() if l.startswith("{")]


def test_reference_arm_line():
    p = _run(["--impl", "reference", "--steps", "3", "--warmup", "3"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert REQUIRED <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    rp = d.get("reference_python")
    if rp is not None:  # the stock reference (oracle/_ref) timed as context
        assert rp["one_core_best"] > 0 and rp["k_processes"]["value"] > 0


def test_reference_arm_under_torchrun_prints_once():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
           "2", "--steps", "3", "--warmup", "3", "--no-reference-python"]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600,
                       env=dict(os.environ, OMP_NUM_THREADS="2"))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_bench_without_gpu_fails_loudly():
    """The GPU arm must not fall back to the CPU: without CUDA it exits non-zero."""
    pytest.importorskip("torch")
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = _run(["--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"], timeout=300)
    assert p.returncode != 0
    assert not _json_lines(p.stdout)


def test_reference_arm_never_loads_the_product_library():
    """The reference arm (and its input generation) runs on the oracle only: no
    libbq.so in the process after a full run."""
    code = ("import sys; sys.argv=['bench.py','--impl','reference','--steps','3','--warmup','3',"
            "'--no-reference-python']; "
            "sys.path.insert(0, %r); import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "assert 'libbq.so' not in maps, 'libbq.so loaded'; assert 'liboracle' in maps" % ROOT)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600,
                       env=dict(os.environ, OMP_NUM_THREADS="2"))
    assert p.returncode == 0, p.stderr[-2000:]
    assert len(_json_lines(p.stdout)) == 1


def test_reference_arm_gpus_flag_reports_world():
    p = _run(["--impl", "reference", "--gpus", "4", "--steps", "3", "--warmup", "3", "--no-reference-python"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 4
