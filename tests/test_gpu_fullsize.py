"""Parity at BASELINE.json's full sizes (configs 2-5), on the B200.

C2 and C3 are compared bit for bit, whole, against the oracle's multi-threaded
C port of the reference algorithms (itself pinned to reference-generated
fixtures in test_oracle.py).  C4 is compared whole against the oracle's
restatement of runmerge.cdom_threshold.  C5 (256 GiB, eight 32 GiB waves) is
checked through size-independent properties -- majority over an odd N is
self-dual, so theta_256(NOT B) = NOT theta_256(B) -- plus oracle windows in
every wave.  The counting identity sum_T popcount(theta_T) = sum_i popcount(B_i)
checks C2 across all 64 thresholds.  On top, windows of every full-size result
are compared with the REFERENCE's own outputs on those exact inputs
(tests/golden/baseline.npz: C2 first / middle / last windows at every T, C3 and
C5 first / last windows, C4's first 2^20 bits at T = 10, 20, 50)."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SEED = 1402


def _baseline():
    """Reference-run outputs on windows of these exact inputs (make_golden.py baseline_cases)."""
    import json
    import os

    z = np.load(os.path.join(GOLDEN, "baseline.npz"))
    return z, json.loads(str(z["meta"]))


def _check_reference_windows(prefix, got_words_at):
    """Every reference window fixture named prefix*: got_words_at(meta) -> words."""
    z, meta = _baseline()
    names = [k for k in meta if k.startswith(prefix)]
    assert names
    for k in names:
        assert np.array_equal(got_words_at(meta[k]), z[k]), k


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def _rows(lib, n, w0, nw, q16s):
    data = torch.empty((n, nw), dtype=torch.int64, device="cuda")
    q = np.ascontiguousarray(q16s, dtype=np.uint32)
    assert lib.bq_gen_bernoulli_rows(SEED, 0, n, q.ctypes.data, w0, nw, data.data_ptr(), nw,
                                     torch.cuda.current_stream().cuda_stream) == 0
    return data


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def _popcount(words: np.ndarray) -> int:
    return int(np.unpackbits(words.view(np.uint8)).sum())


def test_c2_full_size_bit_exact(bq):
    """Config 2 whole: N=64 x 2^22 words (2 GiB), densities in [0.01, 0.5], every T
    of the sweep against the oracle port; OR / AND against torch reductions;
    theta_{T+1} within theta_T; the counting identity over all 64 thresholds."""
    lib = bq._lib.load()
    n, nw = 64, 1 << 22
    data = _rows(lib, n, 0, nw, [lib.bq_gen_density_q16(SEED, i, 655, 32768) for i in range(n)])
    q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
    host = _host(data).reshape(n, nw)
    rows = [host[i] for i in range(n)]
    total_pc, prev, sweep = 0, None, {}
    for t in range(1, n + 1):
        out, pc = q.threshold(t)
        total_pc += int(pc.item())
        if prev is not None:
            assert not torch.any(out[:nw] & ~prev).item(), f"theta_{t} not within theta_{t - 1}"
        if t in (1, 2, 16, 32, 64):
            exp = O.threshold_port(rows, 64 * nw, t)
            got = _host(out[:nw])
            assert np.array_equal(got, exp), t
            assert int(pc.item()) == _popcount(exp)
            sweep[t] = got
        if t == 1:
            ref = data[0].clone()
            for i in range(1, n):
                ref |= data[i]
            assert torch.equal(out[:nw], ref)
        if t == n:
            ref = data[0].clone()
            for i in range(1, n):
                ref &= data[i]
            assert torch.equal(out[:nw], ref)
        prev = out[:nw].clone()
    assert total_pc == sum(_popcount(r) for r in rows)  # each set bit counted once per T <= its count
    # the reference's own answers on the first, middle and last 2^12-word windows, every T
    _check_reference_windows("c2_", lambda m: sweep[m["t"]][m["w0"]:m["w0"] + m["nw"]])
    q.close()


def test_c3_full_size_bit_exact(bq):
    """Config 3 whole: N=256 x 2^20 words (2 GiB), p=0.05, count in [2, 10]."""
    lib = bq._lib.load()
    n, nw = 256, 1 << 20
    data = _rows(lib, n, 0, nw, [3277] * n)
    q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
    acc = [2 <= k <= 10 for k in range(n + 1)]
    out, pc = q.symmetric(acc)
    host = _host(data).reshape(n, nw)
    exp = O.symmetric_port([host[i] for i in range(n)], 64 * nw, acc)
    got = _host(out[:nw])
    assert np.array_equal(got, exp)
    assert int(pc.item()) == _popcount(exp)
    _check_reference_windows("c3_", lambda m: got[m["w0"]:m["w0"] + m["nw"]])
    q.close()


def _markov(lib, i, r):
    cap = (r // 64) // 8 + 4096
    while True:
        buf = np.empty(cap, dtype=np.uint64)
        k = ctypes.c_uint64(0)
        rc = lib.bq_gen_markov_rle(SEED, i, r, 256.0, 12544.0, buf.ctypes.data, cap, ctypes.byref(k))
        if rc == 0:
            return buf[: k.value].copy()
        cap *= 2


def test_c4_full_size_bit_exact(bq):
    """Config 4 whole: N=1024 EWAH streams of r=2^30 bits (2.4 GB compressed),
    T=50, through K4 (first evaluation) and K4s (tile-sliced layout), against the
    oracle's cdom sweep (single-threaded, as the reference)."""
    lib = bq._lib.load()
    n, r, t = 1024, 1 << 30, 50
    nw = r // 64
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(16) as ex:  # ctypes releases the GIL
        streams = list(ex.map(lambda i: _markov(lib, i, r), range(n)))
    d = [torch.from_numpy(s.view(np.int64)).cuda() for s in streams]
    q = bq.RleQuery(d, r)
    st = {}
    exp = O.cdom_threshold(streams, r, t, stats=st)
    z, _ = _baseline()
    assert np.array_equal(exp[: 1 << 14], z["c4_t50"])  # the reference's answer on the first 2^20 bits
    for _ in range(2):
        out, pc = q.threshold(t)
        assert np.array_equal(_host(out[:nw]), exp)
        assert int(pc.item()) == _popcount(exp)
    assert q.layout_stats[0] > 0
    assert q.sweep_stats(t) == st  # K8: the sweep's segments / heap_pops / branches at full size


def test_c5_full_size_properties(bq):
    """Config 5 whole (N=511, r=2^32 bits, p=0.5, T=256: 256 GiB) in eight 32 GiB
    waves: majority over odd N is self-dual, theta_256(NOT B) = NOT theta_256(B),
    checked on every word; two 4096-word windows per wave against the oracle."""
    lib = bq._lib.load()
    n, total, t = 511, 1 << 26, 256
    wave = 1 << 23
    data = torch.empty((n, wave), dtype=torch.int64, device="cuda")
    q16 = np.full(n, 32768, dtype=np.uint32)
    rng = np.random.default_rng(0)
    total_pc = 0
    for w0 in range(0, total, wave):
        assert lib.bq_gen_bernoulli_rows(SEED, 0, n, q16.ctypes.data, w0, wave, data.data_ptr(), wave,
                                         torch.cuda.current_stream().cuda_stream) == 0
        q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * wave)
        out, pc = q.threshold(t)
        total_pc += int(pc.item())
        for a in (0, int(rng.integers(1, wave // 4096)) * 4096):
            win = [_host(data[i, a:a + 4096]) for i in range(n)]
            assert np.array_equal(_host(out[a:a + 4096]), O.threshold_port(win, 64 * 4096, t)), (w0, a)
        z, meta = _baseline()
        for k, m in meta.items():  # the reference's answers on the first and last 2^10 words
            if k.startswith("c5_") and w0 <= m["w0"] < w0 + wave:
                a = m["w0"] - w0
                assert np.array_equal(_host(out[a:a + m["nw"]]), z[k]), k
        res = out[:wave].clone()
        q.close()
        data.bitwise_not_()  # r is a multiple of 64: no tail bits to mask
        q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * wave)
        out2, _ = q.threshold(t)
        assert torch.equal(out2[:wave], ~res), w0
        q.close()
    assert abs(total_pc / (64.0 * total) - 0.5) < 0.01


def test_c4_full_size_low_t_and_symmetric(bq):
    """Config 4's streams at full size with T=5 (most words undecided by the fills:
    phase C reads literal words in nearly every tile) and a symmetric interval
    [3, 40], through K4s, against the oracle's cdom sweeps."""
    lib = bq._lib.load()
    n, r = 1024, 1 << 30
    nw = r // 64
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(16) as ex:
        streams = list(ex.map(lambda i: _markov(lib, i, r), range(n)))
    d = [torch.from_numpy(s.view(np.int64)).cuda() for s in streams]
    q = bq.RleQuery(d, r)
    q.threshold(50)  # first evaluation (K4); the next ones run on the tile-sliced layout
    out, pc = q.threshold(5)
    exp = O.cdom_threshold(streams, r, 5)
    assert np.array_equal(_host(out[:nw]), exp)
    assert int(pc.item()) == _popcount(exp)
    acc = [3 <= k <= 40 for k in range(n + 1)]
    out, pc = q.symmetric(acc)
    exp = O.cdom_symmetric(streams, r, acc)
    assert np.array_equal(_host(out[:nw]), exp)
    assert int(pc.item()) == _popcount(exp)
    # thresholds where phase C runs in most tiles: whole results against the oracle's
    # cdom sweep, and the first 2^20 bits against the reference's own cdom_threshold
    z, _ = _baseline()
    for t in (10, 20, 30):
        out, pc = q.threshold(t)
        got = _host(out[:nw])
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(got, exp), t
        assert int(pc.item()) == _popcount(exp), t
        if t in (10, 20):
            assert np.array_equal(got[: 1 << 14], z[f"c4_t{t}"]), t
    q.close()
