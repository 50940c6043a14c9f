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
    c5 = d["c5_strong_scaling"]
    assert c5["scaling"] == "strong" and c5["n_gpus"] == 1 and c5["waves_per_rank"] == 8
    assert c5["value"] > 0 and c5["input_bytes"] == 511 * (1 << 26) * 8 and c5["popcount"] > 0


def test_c4_line_contract():
    d = _bench("--workload", "c4", "--steps", "5", "--warmup", "3", "--no-e2e")
    assert {"metric", "value", "roofline", "cpu_baseline", "gpu_launches", "clocks"} <= set(d)
    assert d["matches_oracle_window"] and d["popcount"] > 0
    f = d["fresh_query_ms"]
    assert f["k3_directory"] > 0 and f["k4_first_eval"] > 0 and f["total"] >= f["k3_directory"]
    assert d["repeated_query"]["layout"]["markers"] > 0 and d["repeated_query"]["mean_launch_ms"] > 0
    assert d["roofline"]["frac"] < 1.2  # input bytes over the fresh query: never above the HBM peak


@pytest.mark.parametrize("workload", ["c2", "c4"])
def test_two_ranks_under_torchrun(workload):
    """The multi-rank flow (word-range shards, popcount all-reduce, max-over-ranks
    timing, rank 0 prints) with two ranks sharing the one GPU over gloo; a
    functional check of the N > 1 path, not a measurement."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--workload", workload, "--gpus",
           "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1"]
    env = dict(os.environ, BQ_BENCH_BACKEND="gloo", BQ_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="2")
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and "clocks" in d
    if workload == "c2":
        assert d["e2e"]["matches_device_result"]
    else:
        assert d["matches_oracle_window"] and d["popcount"] > 0


def test_gpus_flag_launches_its_own_ranks():
    """``bench.py --gpus 2`` outside torchrun starts two ranks itself (here sharing
    the one GPU over gloo: a functional check, not a measurement) and rank 0 prints
    one line with n_gpus = 2, including the C5 strong-scaling fields."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, BQ_BENCH_BACKEND="gloo", BQ_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="2")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                        "3", "--e2e-steps", "1"], capture_output=True, text=True, cwd=ROOT, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["matches_device_result"]
    c5 = d["c5_strong_scaling"]
    assert c5["n_gpus"] == 2 and c5["waves_per_rank"] == 4 and c5["input_bytes"] == 511 * (1 << 26) * 8


def test_frows_line():
    """The §8(f) rows and the drop-in path, each with its bytes and an exactness check."""
    d = _bench("--workload", "frows", "--steps", "5", "--warmup", "3")
    rows = d["rows"]
    for k in ("binop_and", "binop_or", "binop_xor", "binop_andnot", "binop_not", "encode_dense",
              "encode_c2_t16_result", "nvrtc_ssum_64_32", "count_kernel_t32_same_query"):
        assert rows[k]["median_ms"] > 0 and rows[k]["gbs"] > 0, k
    assert rows["binop_matches_torch"] and rows["encode_matches_oracle"] and rows["nvrtc_matches_count_kernel"]
    if "drop_in_c1" in rows:
        assert rows["drop_in_c1"]["matches_reference"]
