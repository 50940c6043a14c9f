"""The C-ABI multi-device entry bq_shard_threshold (include/bq.h):
one query split by word range into shards whose inputs are separate local
slices, evaluated shard by shard with only the popcount summed.  On this
one-GPU box every shard is placed on device 0 (the code path per device is the
same); the concatenated shard outputs must equal the whole result.  Needs a B200."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


@pytest.mark.parametrize("n,r,t,cuts", [(16, 64 * 10000 + 13, 5, (0, 2048, 6000, 10001)),
                                        (64, 64 * 4096, 32, (0, 1024, 2048, 3072, 4096)),
                                        (7, 64 * 100, 7, (0, 100))])
def test_shard_threshold_tiles_the_result(bq, n, r, t, cuts):
    lib = bq._lib.load()
    nw = (r + 63) // 64
    rng = np.random.default_rng(n * 31 + t)
    host = []
    for i in range(n):
        a = rng.integers(0, 2**63, nw, dtype=np.uint64) | rng.integers(0, 2**63, nw, dtype=np.uint64)
        if r % 64:
            a[-1] &= np.uint64((1 << (r % 64)) - 1)
        host.append(a[: nw - (i % 3) * 7])  # ragged trimmed lengths
    g = len(cuts) - 1
    keep, spans = [], np.zeros((g * n, 2), dtype=np.uint64)
    outs = []
    for s in range(g):
        b, e = cuts[s], cuts[s + 1]
        for i in range(n):
            loc = host[i][b:e] if b < host[i].size else host[i][:0]
            d = torch.from_numpy(np.ascontiguousarray(loc).view(np.int64)).cuda() if loc.size else \
                torch.zeros(2, dtype=torch.int64, device="cuda")
            keep.append(d)
            spans[s * n + i] = (d.data_ptr() if loc.size else 0, loc.size)
        outs.append(torch.empty(max(e - b, 2), dtype=torch.int64, device="cuda"))
    devices = (ctypes.c_int * g)(*([0] * g))
    wb = (ctypes.c_uint64 * g)(*cuts[:-1])
    we = (ctypes.c_uint64 * g)(*cuts[1:])
    optr = (ctypes.c_void_p * g)(*[o.data_ptr() for o in outs])
    pc = ctypes.c_ulonglong(0)
    rc = lib.bq_shard_threshold(g, devices, spans.ctypes.data, n, r, wb, we, t, optr, ctypes.byref(pc), None)
    assert rc == 0, lib.bq_last_error()
    got = np.concatenate([outs[s][: cuts[s + 1] - cuts[s]].cpu().numpy().view(np.uint64) for s in range(g)])
    exp = O.scan_count(host, r, t)
    assert np.array_equal(got, exp)
    assert pc.value == int(np.unpackbits(exp.view(np.uint8)).sum())


def test_shard_threshold_contract(bq):
    lib = bq._lib.load()
    devices = (ctypes.c_int * 1)(0)
    wb = (ctypes.c_uint64 * 1)(1)  # odd start
    we = (ctypes.c_uint64 * 1)(10)
    spans = np.zeros((1, 2), dtype=np.uint64)
    out = torch.empty(16, dtype=torch.int64, device="cuda")
    optr = (ctypes.c_void_p * 1)(out.data_ptr())
    assert lib.bq_shard_threshold(1, devices, spans.ctypes.data, 1, 640, wb, we, 1, optr, None, None) == -1


@pytest.mark.parametrize("n,r", [(1, 64 * 7 + 5), (9, 64 * 3000 + 1), (130, 64 * 2048)])
def test_one_shot_forms(bq, n, r):
    """bq_threshold_u64 / bq_symmetric_u64 (create + evaluate + destroy in one call)
    against the oracle's ScanCount (counters.py:46-83), ragged trimmed inputs."""
    lib = bq._lib.load()
    nw = (r + 63) // 64
    rng = np.random.default_rng(n + r)
    host, keep = [], []
    spans = np.zeros((n, 2), dtype=np.uint64)
    for i in range(n):
        a = rng.integers(0, 2**63, nw, dtype=np.uint64) & rng.integers(0, 2**63, nw, dtype=np.uint64)
        if r % 64:
            a[-1] &= np.uint64((1 << (r % 64)) - 1)
        a = a[: max(0, nw - (i % 4) * 3)]
        host.append(a)
        d = torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda() if a.size else None
        keep.append(d)
        spans[i] = (d.data_ptr() if a.size else 0, a.size)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device="cuda")
    pc = torch.zeros(1, dtype=torch.int64, device="cuda")
    for t in sorted({1, max(1, n // 3), n}):
        pc.zero_()
        torch.cuda.synchronize()
        rc = lib.bq_threshold_u64(spans.ctypes.data, n, r, t, out.data_ptr(), pc.data_ptr(), None)
        assert rc == 0, lib.bq_last_error()
        exp = O.scan_count(host, r, t)
        assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp), t
        assert int(pc.item()) == int(np.unpackbits(exp.view(np.uint8)).sum())
    acc = np.array([k % 3 == 1 for k in range(n + 1)], dtype=np.uint8)
    pc.zero_()
    torch.cuda.synchronize()
    rc = lib.bq_symmetric_u64(spans.ctypes.data, n, r, acc.ctypes.data, out.data_ptr(), pc.data_ptr(), None)
    assert rc == 0, lib.bq_last_error()
    exp = O.scan_count_symmetric(host, r, [bool(x) for x in acc])
    assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp)
    assert int(pc.item()) == int(np.unpackbits(exp.view(np.uint8)).sum())
    # the threshold contract of the one-shot form is the query's: t outside [1, n] is an InputError
    assert lib.bq_threshold_u64(spans.ctypes.data, n, r, n + 1, out.data_ptr(), None, None) != 0
