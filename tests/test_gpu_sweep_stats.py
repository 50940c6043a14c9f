"""K8: cdom's sweep counters (segments, heap_pops, branches; runmerge.py:237-240,
:296-298) recomputed on the device, against the reference's own dicts (golden
fixtures and the C4-prefix baseline) and the oracle's restated sweep on
adversarial non-canonical streams.  Needs a B200."""

from __future__ import annotations

import ctypes
import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RLE = load_golden("rle")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def dev(bq, arrs):
    out = []
    for a in arrs:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        t = torch.from_numpy(a.view(np.int64)).cuda() if a.size else torch.zeros(1, dtype=torch.int64, device="cuda")
        out.append(bq.DeviceRleBitmap(t, 0, a.size))
    return out


@pytest.mark.parametrize("case", RLE, ids=lambda c: c.id)
def test_stats_match_reference_dicts(bq, case):
    """Reference RleBitmap mirrors in, the reference's stats dict out (key for key)."""
    ins = [bq.RleBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    st = {}
    if case.meta["kind"] == "cdom_threshold":
        bq.cdom_threshold(ins, case.meta["t"], stats=st)
    else:
        bq.cdom_symmetric(ins, bq.SymmetricSpec(tuple(bool(x) for x in case.meta["accept"])), stats=st)
    assert st == case.meta["stats"]


def _marker(bit, run, dirty):
    return (dirty << 33) | (run << 1) | bit


def _stream(rng, total):
    """A valid but non-canonical stream: empty markers, same-bit fills split across
    markers, literal groups back to back, fills spanning tiles, coverage short of
    total (implicit zero tail) or exact."""
    out, cov = [], 0
    target = total if rng.random() < 0.5 else int(total * rng.random())
    while cov < target:
        kind = rng.random()
        if kind < 0.1:
            out.append(_marker(int(rng.integers(2)), 0, 0))
            continue
        room = target - cov
        run = int(min(room, rng.choice([0, 1, 2, 5, 40, 700, 3000]) if kind < 0.9 else room))
        dirty = int(min(room - run, rng.choice([0, 0, 1, 2, 3, 17])))
        edge = 1024 - (cov + run) % 1024  # end the fill or the literal group on a tile boundary
        if kind < 0.25 and edge <= room - run:
            if rng.random() < 0.5:
                run, dirty = run + edge, 0
            elif edge <= 40:
                dirty = edge
        bit = int(rng.integers(2))
        out.append(_marker(bit, run, dirty))
        for _ in range(dirty):
            w = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(2))
            out.append(w if rng.random() < 0.8 else (1 << 64) - 1)
        cov += run + dirty
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("seed", range(16))
def test_stats_adversarial_streams_vs_oracle(bq, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([2, 3, 7, 33, 130, 300]))
    total = int(rng.choice([1, 5, 1023, 1024, 1025, 3000, 4100]))
    r = 64 * total
    streams = [_stream(rng, total) for _ in range(n)]
    if seed % 3 == 0:
        streams[0] = np.zeros(0, dtype=np.uint64)  # an empty stream: all implicit tail
    q = bq.RleQuery(dev(bq, streams), r)
    for t in sorted({2, max(2, n // 4), max(2, n // 2), n - 1, min(n - 1, 150)}):
        if not 1 < t < n:
            continue
        exp = {}
        O.cdom_threshold(streams, r, t, stats=exp)
        assert q.sweep_stats(t) == exp, t
    exp = {}
    O.cdom_symmetric(streams, r, [k % 3 == 1 for k in range(n + 1)], stats=exp)
    assert q.sweep_stats(0) == exp


def test_stats_c4_prefix_vs_reference(bq):
    """The C4 Markov streams over their first 2^20 bits, T in {5, 10, 20, 50}: the
    reference's own cdom stats (tests/golden/baseline.npz)."""
    import os

    from conftest import GOLDEN

    base = np.load(os.path.join(GOLDEN, "baseline.npz"))
    meta = json.loads(str(base["meta"]))
    lib = bq._lib.load()
    n, r = 1024, 1 << 20
    streams = []
    for i in range(n):
        cap = 2 * (r // 64) + 64
        buf = np.empty(cap, dtype=np.uint64)
        k = ctypes.c_uint64(0)
        assert lib.bq_gen_markov_rle(1402, i, r, 256.0, 12544.0, buf.ctypes.data, cap, ctypes.byref(k)) == 0
        streams.append(buf[: k.value].copy())
    ins = [bq.RleBitmap(s.tolist(), r) for s in streams]
    for t in (5, 10, 20, 50):
        st = {}
        bq.cdom_threshold(ins, t, stats=st)
        assert st == meta[f"c4_t{t}"]["stats"], t


def test_stats_untouched_where_the_reference_skips_the_sweep(bq):
    ins = [bq.RleBitmap([_marker(1, 3, 0)], 64 * 3), bq.RleBitmap([_marker(0, 1, 1), 5], 64 * 3)]
    for t in (1, 2):  # T = 1 -> wide_or, T = N -> wide_and (runmerge.py:203-206)
        st = {"x": 1}
        bq.cdom_threshold(ins, t, stats=st)
        assert st == {"x": 1}
    st = {}
    bq.cdom_symmetric([bq.RleBitmap([], 0)] * 2, bq.SymmetricSpec.parity(2), stats=st)
    assert st == {}  # r = 0 (:257-258)


def test_stats_need_the_whole_range(bq):
    streams = [np.array([_marker(1, 2048, 0)], dtype=np.uint64)] * 3
    q = bq.RleQuery(dev(bq, streams), 64 * 2048, word_range=(1024, 2048))
    with pytest.raises(bq.InputError):
        q.sweep_stats(2)
