"""The CUDA path against the REFERENCE's own outputs on BASELINE.json's seeded
inputs (tests/golden/baseline.npz, written by make_golden.py baseline_cases,
which runs reference counters.scan_count / scan_count_symmetric, looped,
csv_threshold, wide_or / wide_and, CircuitLibrary and runmerge.cdom_threshold):

* C1 in full (N=8, r=2^20, T=3);
* C2 windows of 2^12 words x 64 bitmaps (first, middle, last) at every T;
* C3 windows (N=256, accept [2, 10]), first and last;
* C5 windows (N=511, T=256), first and last;
* C4's 1024 Markov streams over their first 2^20 bits at T = 5, 10, 20, 50, on
  both K4 paths (per-stream and tile-sliced).

Inputs are generated on the device by the product generator (csrc/bq_gen.h,
pinned by kat.json), so the comparison covers exactly what bench.py measures.
The full-size runs (test_gpu_fullsize.py) check the same windows inside the
whole 2 GiB / 256 GiB / 2^30-bit results.  Needs a B200."""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

Z = np.load(os.path.join(GOLDEN, "baseline.npz"))
META = json.loads(str(Z["meta"]))
WINDOWS = sorted(k for k in META if not k.startswith("c4"))


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def _rows(lib, n, w0, nw, q16):
    data = torch.empty((n, nw), dtype=torch.int64, device="cuda")
    q = np.ascontiguousarray(q16 if isinstance(q16, list) else [q16] * n, dtype=np.uint32)
    assert lib.bq_gen_bernoulli_rows(1402, 0, n, q.ctypes.data, w0, nw, data.data_ptr(), nw,
                                     torch.cuda.current_stream().cuda_stream) == 0
    return data


def _popcount(words) -> int:
    return int(np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8)).sum())


@pytest.mark.parametrize("name", WINDOWS)
def test_uncompressed_configs_match_reference(bq, name):
    lib = bq._lib.load()
    m = META[name]
    n, w0, nw = m["n"], m["w0"], m["nw"]
    data = _rows(lib, n, w0, nw, m["q16"])
    q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
    if name.startswith("c3"):
        out, pc = q.symmetric(bq.SymmetricSpec.interval(n, 2, 10))
    else:
        out, pc = q.threshold(m["t"])
    got = out[:nw].cpu().numpy().view(np.uint64)
    assert np.array_equal(got, Z[name]), name
    assert int(pc.item()) == m["card"]
    q.close()


def _markov_device(lib, n, r):
    streams = []
    for i in range(n):
        cap = max(4096, r // 64 // 4)
        buf = np.empty(cap, dtype=np.uint64)
        k = ctypes.c_uint64(0)
        assert lib.bq_gen_markov_rle(1402, i, r, 256.0, 12544.0, buf.ctypes.data, cap, ctypes.byref(k)) == 0
        streams.append(torch.from_numpy(buf[: k.value].copy().view(np.int64)).cuda())
    return streams


@pytest.mark.parametrize("sliced", ["0", "1"], ids=["per_stream", "sliced"])
def test_c4_prefix_matches_reference(bq, sliced, monkeypatch):
    monkeypatch.setenv("BQ_RLE_SLICED", sliced)
    lib = bq._lib.load()
    r = 1 << 20
    d = _markov_device(lib, 1024, r)
    q = bq.RleQuery([bq.DeviceRleBitmap(t, r, t.numel()) for t in d], r)
    for t in (5, 10, 20, 50):
        out, pc = q.threshold(t)
        got = out[: r // 64].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, Z[f"c4_t{t}"]), t
        assert int(pc.item()) == META[f"c4_t{t}"]["card"] == _popcount(got)
    q.close()


def test_c4_prefix_drop_in_rle_result(bq):
    """Through the drop-in cdom_threshold with device streams: the result is the
    uncompressed device bitmap; re-encoding it on the device (K7) gives exactly the
    reference's RleBitmap length (rle_out_len)."""
    lib = bq._lib.load()
    r = 1 << 20
    d = [bq.DeviceRleBitmap(t, r, t.numel()) for t in _markov_device(lib, 1024, r)]
    for t in (10, 20):
        res = bq.cdom_threshold(d, t)
        words = res.data[: r // 64]
        assert np.array_equal(words.cpu().numpy().view(np.uint64), Z[f"c4_t{t}"])
        enc = bq.api.encode_device(words, r)
        assert enc.size == META[f"c4_t{t}"]["rle_out_len"]
