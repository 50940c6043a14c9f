"""The device canonical RLE encoder K7 (bq_rle_encode_device; RleBuilder /
compress, reference bitmaps.py:351-414) against the oracle's restatement, which
is pinned to the reference's own compress in test_oracle.py.  Covers long
literal runs (a whole dense bitmap is one marker and its literals), leading
literal runs, alternating fills, trimmed inputs (implicit zero tail) and r % 64
!= 0.  Needs a B200."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1402_4073_b200 import _lib

    return _lib.load()


def _words(kind, nw, rng):
    if kind == "dense":
        return rng.integers(1, 2**63, nw, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    if kind == "sparse":
        w = np.zeros(nw, dtype=np.uint64)
        idx = rng.integers(0, nw, max(1, nw // 50))
        w[idx] = rng.integers(1, 2**63, idx.size, dtype=np.uint64)
        return w
    if kind == "fills":
        return np.where(rng.random(nw) < 0.5, np.uint64(0), np.uint64(2**64 - 1)).astype(np.uint64)
    if kind == "mixed":
        choice = rng.integers(0, 3, nw)
        vals = rng.integers(1, 2**63, nw, dtype=np.uint64)
        return np.where(choice == 0, np.uint64(0), np.where(choice == 1, np.uint64(2**64 - 1), vals)).astype(np.uint64)
    if kind == "runs":
        w = np.zeros(nw, dtype=np.uint64)
        pos = 0
        while pos < nw:
            ln = int(rng.integers(1, 300))
            w[pos:pos + ln] = [np.uint64(0), np.uint64(2**64 - 1), np.uint64(0x55)][int(rng.integers(0, 3))]
            pos += ln
        return w
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["dense", "sparse", "fills", "mixed", "runs"])
@pytest.mark.parametrize("nw,trim,tail", [(1, 0, 0), (37, 0, 5), (4096, 100, 0), (1 << 20, 0, 17), (3001, 3001, 0)])
def test_device_encoder_matches_compress(lib, kind, nw, trim, tail):
    rng = np.random.default_rng(nw + trim + tail + len(kind))
    r = 64 * nw - (64 - tail if tail else 0)
    w = _words(kind, nw, rng)
    if tail:
        w[-1] &= np.uint64((1 << tail) - 1)
    valid = nw - trim
    dw = torch.from_numpy(w.view(np.int64)).cuda()
    cap = nw + 2
    out = torch.empty(cap, dtype=torch.int64, device="cuda")
    n_out = ctypes.c_uint64(0)
    rc = lib.bq_rle_encode_device(dw.data_ptr(), valid, r, out.data_ptr(), cap, ctypes.byref(n_out),
                                  torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.bq_last_error()
    got = out[: n_out.value].cpu().numpy().view(np.uint64)
    exp = O.rle_compress(w[:valid], r)
    assert np.array_equal(got, exp)
