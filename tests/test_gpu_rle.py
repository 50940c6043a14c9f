"""Parity of the device RLE path (K3 directory + K4 tile decode-and-count) with
the reference cdom algorithms and decoder.  Needs a B200."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import load_golden, padded
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RLE = load_golden("rle")
CODEC = load_golden("codec")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


@pytest.fixture(autouse=True, params=["0", "1"], ids=["per_stream", "sliced"])
def rle_layout(request, monkeypatch):
    """Run every case on both K4 paths: the per-stream walk (BQ_RLE_SLICED=0) and the
    tile-sliced layout built at the first evaluation (BQ_RLE_SLICED=1)."""
    monkeypatch.setenv("BQ_RLE_SLICED", request.param)
    return request.param


def dev(arrs):
    out = []
    for a in arrs:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        t = torch.from_numpy(a.view(np.int64)).cuda() if a.size else torch.zeros(1, dtype=torch.int64, device="cuda")
        out.append(bq_stream(t, a.size))
    return out


def bq_stream(t, n):
    import paper_1402_4073_b200 as bq

    return bq.DeviceRleBitmap(t, 0, n)


def host(t, nw):
    return t[:nw].cpu().numpy().view(np.uint64)


def popcount(words):
    return int(np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8)).sum())


def markov(lib, seed, i, r, m1, m0):
    cap = max(1024, (r // 64) * 2 + 16)
    out = np.empty(cap, dtype=np.uint64)
    n = ctypes.c_uint64(0)
    assert lib.bq_gen_markov_rle(seed, i, r, m1, m0, out.ctypes.data, cap, ctypes.byref(n)) == 0
    return out[: n.value].copy()


@pytest.mark.parametrize("case", RLE, ids=lambda c: c.id)
def test_cdom_golden(bq, case):
    q = bq.RleQuery(dev(case.inputs), case.r)
    if case.meta["kind"] == "cdom_threshold":
        out, pc = q.threshold(case.meta["t"])
    else:
        out, pc = q.symmetric(case.meta["accept"])
    nw = (case.r + 63) // 64
    exp = padded(np.array(case.meta["uncompressed"], dtype=np.uint64), case.r)
    assert np.array_equal(host(out, nw), exp)
    assert int(pc.item()) == popcount(exp)


@pytest.mark.parametrize("case", RLE[::2], ids=lambda c: c.id)
def test_cdom_golden_dropin(bq, case):
    """Reference-style RleBitmap in -> canonical RleBitmap out, word for word."""
    ins = [bq.RleBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    if case.meta["kind"] == "cdom_threshold":
        got = bq.cdom_threshold(ins, case.meta["t"])
        assert bq.scan_count(ins, case.meta["t"]).words == case.out.tolist()  # RLE in -> RLE out
    else:
        got = bq.cdom_symmetric(ins, bq.SymmetricSpec(tuple(bool(x) for x in case.meta["accept"])))
    assert isinstance(got, bq.RleBitmap)
    assert got.words == case.out.tolist()
    assert got.bit_length == case.r


@pytest.mark.parametrize("case", CODEC, ids=lambda c: c.id)
def test_device_decoder_codec(bq, case):
    if case.meta["kind"] == "compress":
        stream, expect = case.out, padded(case.inputs[0], case.r)
    else:
        stream, expect = case.inputs[0], padded(case.out, case.r)
    rb = bq.RleBitmap(stream.tolist(), case.r)
    if case.meta.get("status") == "format_error":
        with pytest.raises(bq.FormatError):
            bq.decompress(rb)
        return
    got = bq.decompress(rb)
    assert isinstance(got, bq.UncompressedBitmap)
    assert np.array_equal(padded(np.array(got.words, dtype=np.uint64), case.r), expect)


@pytest.mark.parametrize("n,r,m1,m0", [(1, 64 * 5000, 40.0, 300.0), (7, 64 * 20000 + 3, 256.0, 12544.0),
                                      (64, (1 << 20) + 17, 30.0, 90.0), (300, 1 << 21, 256.0, 12544.0),
                                      (33, 64 * 4096 * 3, 5000.0, 5000.0), (16, 64 * 100, 3.0, 3.0)])
def test_markov_vs_oracle_cdom(bq, n, r, m1, m0):
    lib = bq._lib.load()
    streams = [markov(lib, 77, i, r, m1, m0) for i in range(n)]
    q = bq.RleQuery(dev(streams), r)
    nw = (r + 63) // 64
    for t in sorted({1, 2, 3, max(1, n // 10), max(1, n // 2), n} & set(range(1, n + 1))):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
    for acc in ([k % 2 == 1 for k in range(n + 1)], [k == 0 or 2 <= k <= 4 for k in range(n + 1)]):
        out, pc = q.symmetric(acc)
        exp = O.cdom_symmetric(streams, r, acc)
        assert np.array_equal(host(out, nw), exp)
        assert int(pc.item()) == popcount(exp)


def test_ragged_and_degenerate_streams(bq):
    """Empty streams, short streams (implicit tail), fill_run=0 markers, literal
    all-0/all-1 words, dirty runs across tile boundaries, long one-fills."""
    mk = lambda bit, run, dirty: bit | (run << 1) | (dirty << 33)  # noqa: E731
    r = 64 * 4096 * 3 + 7
    nw = (r + 63) // 64
    rng = np.random.default_rng(3)
    lits = [int(x) for x in rng.integers(1, 2**63, size=40)]
    streams = [
        np.array([], dtype=np.uint64),
        np.array([mk(1, 4090, 10)] + lits[:10], dtype=np.uint64),          # dirty run across tile 0/1
        np.array([mk(0, 0, 2), lits[10], lits[11], mk(1, 9000, 0)], dtype=np.uint64),
        np.array([mk(1, 0, 3), 0, 2**64 - 1, lits[12], mk(0, 4093, 0), mk(1, 2, 5)] + lits[13:18],
                 dtype=np.uint64),
        np.array([mk(1, nw - 1, 0)], dtype=np.uint64),                     # ones to the last full word
        np.array([mk(0, 4095, 1), lits[20], mk(0, 0, 0), mk(0, 0, 1), lits[21]], dtype=np.uint64),
    ]
    q = bq.RleQuery(dev(streams), r)
    n = len(streams)
    for t in range(1, n + 1):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        dec = [O.rle_decompress(s, r) for s in streams]
        assert np.array_equal(exp, O.scan_count(dec, r, t))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_directory_ring_horizon(bq, seed):
    """K3a's staging ring (14 windows of 32 words ahead) and its 4-window chain
    tables: literal groups whose lengths straddle the ring horizon (a restart at the
    next marker) and the group boundary, markers landing on window and group edges,
    streams whose length is not a multiple of 32, and an implicit zero tail."""
    mk = lambda bit, run, dirty: bit | (run << 1) | (dirty << 33)  # noqa: E731
    rng = np.random.default_rng(100 + seed)
    r = 64 * 1024 * 24 + 5
    nw = (r + 63) // 64
    streams = []
    for i in range(24):
        out, covered = [], 0
        while covered < nw - 2000:
            kind = rng.integers(0, 4)
            if kind == 0:  # a literal group around the ring horizon (448 words) or a group edge (128)
                d = int(rng.choice([1, 31, 32, 33, 95, 127, 128, 129, 445, 446, 447, 448, 449, 480, 900]))
            else:
                d = int(rng.integers(0, 4))
            run = int(rng.integers(0, 300))
            d = min(d, nw - covered - run)
            out.append(mk(int(rng.integers(0, 2)) if run else 0, run, d))
            out.extend(int(x) for x in rng.integers(1, 2**63, size=d))
            covered += run + d
        if i % 3 == 0:  # explicit fill to the end; otherwise the implicit zero tail
            out.append(mk(0, nw - covered, 0))
        streams.append(np.array(out, dtype=np.uint64))
    q = bq.RleQuery(dev(streams), r)
    for t in (1, 3, 12, 24):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)


def test_c4_shape_scaled(bq):
    """Config 4 generator (one-runs mean 256, zero-runs 12544, density 0.02) at
    N=1024 and r=2^24 bits, T=50 (the config's T) and T=5,10,20 where the dirty
    literal path is exercised, against the oracle's cdom sweep."""
    lib = bq._lib.load()
    n, r = 1024, 1 << 24
    streams = [markov(lib, 1402, i, r, 256.0, 12544.0) for i in range(n)]
    q = bq.RleQuery(dev(streams), r)
    nw = r // 64
    for t in (5, 10, 20, 50):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)


def test_rle_errors(bq):
    mk = lambda bit, run, dirty: bit | (run << 1) | (dirty << 33)  # noqa: E731
    good = np.array([mk(0, 2, 0)], dtype=np.uint64)
    with pytest.raises(bq.FormatError):
        bq.RleQuery(dev([good, np.array([mk(0, 1, 3), 1, 2], dtype=np.uint64)]), 64 * 10)
    with pytest.raises(bq.FormatError):
        bq.RleQuery(dev([good, np.array([mk(0, 11, 0)], dtype=np.uint64)]), 64 * 10)
    q = bq.RleQuery(dev([good, good]), 64 * 10)
    with pytest.raises(bq.InputError):
        q.threshold(3)
    with pytest.raises(bq.InputError):
        q.symmetric([True, False])


@pytest.mark.parametrize("case", [c for c in CODEC if c.meta["kind"] == "compress"] + RLE[::3], ids=lambda c: c.id)
def test_device_encoder_matches_reference(bq, case):
    """bq_rle_encode_device == the reference's canonical compress (bitmaps.py:407-414)."""
    from paper_1402_4073_b200.api import encode_device

    if case.meta["kind"] == "compress":
        words, expect = case.inputs[0], case.out
    else:
        words, expect = np.array(case.meta["uncompressed"], dtype=np.uint64), case.out
    t = torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint64).view(np.int64)).cuda() if words.size \
        else torch.zeros(0, dtype=torch.int64, device="cuda")
    assert np.array_equal(encode_device(t, case.r), expect)


@pytest.mark.parametrize("seed", range(6))
def test_device_encoder_random(bq, seed):
    from paper_1402_4073_b200.api import compress_words, encode_device

    rng = np.random.default_rng(seed)
    nw = int(rng.integers(1, 20000))
    r = 64 * nw - int(rng.integers(0, 64))
    kinds = rng.integers(0, 3, size=nw)
    words = np.where(kinds == 0, 0, np.where(kinds == 1, np.uint64(2**64 - 1),
                                             rng.integers(1, 2**63, size=nw, dtype=np.uint64))).astype(np.uint64)
    # runs: repeat classes to create long fills
    words = np.repeat(words, rng.integers(1, 6, size=nw))[:nw]
    if r % 64:
        words[-1] &= np.uint64((1 << (r % 64)) - 1)
    cut = int(rng.integers(0, nw + 1))
    t = torch.from_numpy(words[:cut].view(np.int64).copy()).cuda()
    assert encode_device(t, r).tolist() == compress_words(words[:cut], r)


SETOPS = load_golden("setops")


@pytest.mark.parametrize("case", SETOPS, ids=lambda c: c.id + "-" + c.meta["op"])
def test_set_algebra_matches_reference(bq, case):
    """and_/or_/xor/andnot/not_ on the device, both representations (bitmaps.py:438-644)."""
    op = case.meta["op"]
    ua = bq.UncompressedBitmap(case.inputs[0].tolist(), case.bits[0])
    ra = bq.RleBitmap([int(w) for w in case.meta["rle_a"]], case.bits[0])
    if op == "not":
        got_u, got_r = bq.not_(ua, case.r), bq.not_(ra, case.r)
    else:
        ub = bq.UncompressedBitmap(case.inputs[1].tolist(), case.bits[1])
        rb = bq.RleBitmap([int(w) for w in case.meta["rle_b"]], case.bits[1])
        got_u, got_r = bq.binary_op(op, ua, ub), bq.binary_op(op, ra, rb)
    assert got_u.words == case.out.tolist() and got_u.bit_length == case.r
    assert [str(w) for w in got_r.words] == case.meta["rle_out"] and got_r.bit_length == case.r


def test_all_literal_streams_overflow_pools(bq):
    """Uniform random words: every word is a literal, so each tile segment
    (~1025 words per stream) overflows the warp pool (walked from HBM) and every
    output word is undecided (phase C runs in several slot batches)."""
    from oracle import oracle as Or

    rng = np.random.default_rng(11)
    n, r = 40, 64 * 5000 - 9
    nw = (r + 63) // 64
    streams = []
    for i in range(n):
        w = rng.integers(1, 2**63, size=nw, dtype=np.uint64) | np.uint64(1 << 63) if i % 2 else \
            rng.integers(0, 2**64 - 1, size=nw, dtype=np.uint64)
        w[-1] &= np.uint64((1 << (r % 64)) - 1)
        streams.append(Or.rle_compress(Or.trim(w), r))
    q = bq.RleQuery(dev(streams), r)
    for t in (1, 5, 20, 39, 40):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
    acc = [k % 3 == 0 for k in range(n + 1)]
    out, pc = q.symmetric(acc)
    exp = O.cdom_symmetric(streams, r, acc)
    assert np.array_equal(host(out, nw), exp)


def test_phase_c_staging_edges(bq):
    """K4c's staged slices: literal groups that straddle tile ends (the words of a
    slice's last marker past the staged part are read from HBM), more streams than
    the staging table holds (1100 > 1024), streams that end inside a tile, and a
    threshold low enough that nearly every tile reaches phase C."""
    from oracle import oracle as Or

    rng = np.random.default_rng(37)
    n, r = 1100, 64 * 4096 + 21
    nw = (r + 63) // 64
    streams = []
    for i in range(n):
        w = np.zeros(nw, dtype=np.uint64)
        if i % 5 == 0:  # a long literal group across every tile end
            for b in range(1024, nw, 1024):
                lo, hi = b - int(rng.integers(1, 40)), min(nw, b + int(rng.integers(1, 40)))
                w[lo:hi] = rng.integers(1, 2**63, size=hi - lo, dtype=np.uint64)
        elif i % 5 == 1:  # sparse literals and one-fills
            idx = rng.integers(0, nw, size=200)
            w[idx] = rng.integers(1, 2**63, size=idx.size, dtype=np.uint64)
            w[int(rng.integers(0, nw - 300)):][:300] = np.uint64(2**64 - 1)
        elif i % 5 == 2:  # ends inside the second tile (implicit zero tail)
            w[: 1024 + int(rng.integers(1, 900))] = rng.integers(0, 2**64 - 1, size=1, dtype=np.uint64)[0] | np.uint64(5)
        else:  # a few dense windows
            for _ in range(3):
                a = int(rng.integers(0, nw - 64))
                w[a:a + 64] = rng.integers(0, 2**64 - 1, size=64, dtype=np.uint64)
        w[-1] &= np.uint64((1 << (r % 64)) - 1)
        streams.append(Or.rle_compress(Or.trim(w), r))
    q = bq.RleQuery(dev(streams), r)
    for t in (1, 2, 3, 50, 221):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
    acc = [k % 2 == 1 for k in range(n + 1)]
    out, pc = q.symmetric(acc)
    assert np.array_equal(host(out, nw), O.cdom_symmetric(streams, r, acc))


def test_heavy_words_and_bank_skewed_events(bq):
    """K4s phase C's warp path (words with >= 128 literal words) next to its thread
    path in the same tiles, and event lists skewed onto a few shared-memory banks
    (literal words only at positions = 0 mod 32, so every literal start / end event
    falls in banks 0 and 1 and the bank arrangement cannot spread them)."""
    from oracle import oracle as Or

    rng = np.random.default_rng(23)
    n, r = 300, 64 * 2500 + 13
    nw = (r + 63) // 64
    streams = []
    for i in range(n):
        if i < 200:  # dense random words: every word a literal
            w = rng.integers(0, 2**64 - 1, size=nw, dtype=np.uint64)
        else:  # literals at multiples of 32, runs of ones in between for some streams
            w = np.zeros(nw, dtype=np.uint64)
            w[::32] = rng.integers(1, 2**63, size=len(w[::32]), dtype=np.uint64)
            if i % 3 == 0:
                w[5::64] = np.uint64(2**64 - 1)
        w[-1] &= np.uint64((1 << (r % 64)) - 1)
        streams.append(Or.rle_compress(Or.trim(w), r))
    q = bq.RleQuery(dev(streams), r)
    for t in (1, 100, 150, 201, 300):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
    for acc in ([bool(x) for x in rng.integers(0, 2, n + 1)],  # > 64 breakpoints: per-bit decisions
                [k % 2 == 1 for k in range(n + 1)],
                [90 <= k <= 110 for k in range(n + 1)]):
        out, pc = q.symmetric(acc)
        exp = O.cdom_symmetric(streams, r, acc)
        assert np.array_equal(host(out, nw), exp)
        assert int(pc.item()) == popcount(exp)


def test_repeated_dropin_calls_reuse_the_prepared_query(bq):
    """Immutable inputs: the second cdom call on the same objects reuses the
    query (and its K3 directory) and returns the identical result."""
    from paper_1402_4073_b200.api import QUERIES

    case = RLE[0]
    ins = [bq.RleBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    QUERIES.clear()
    first = bq.cdom_threshold(ins, 1)
    n_cached = len(QUERIES._d)
    second = bq.cdom_threshold(ins, 1)
    assert first.words == second.words
    assert len(QUERIES._d) == n_cached == 1


def test_sliced_layout_is_built_at_the_second_evaluation(bq, monkeypatch):
    """Default policy: the first evaluation walks the per-stream layout, the second
    builds the tile-sliced layout (directory_bytes grows) and both agree with the oracle."""
    monkeypatch.delenv("BQ_RLE_SLICED", raising=False)
    lib = bq._lib.load()
    n, r = 96, 1 << 20
    streams = [markov(lib, 77, i, r, 64.0, 900.0) for i in range(n)]
    q = bq.RleQuery(dev(streams), r)
    nw = r // 64
    before = q.directory_bytes
    for k, t in enumerate((3, 3, 7, 50)):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        assert np.array_equal(host(out, nw), exp), (k, t)
        assert int(pc.item()) == popcount(exp)
        if k == 0:
            assert q.directory_bytes == before
    assert q.directory_bytes > before


@pytest.mark.parametrize("acc_kind", ["zero_accepted", "zero_rejected"])
def test_constant_tiles_of_sparse_streams(bq, acc_kind):
    """Sparse streams leave whole tiles with no word able to change the count-0
    answer (the constant-tile path of phase B); with count 0 accepted those tiles
    are all ones.  Ragged r so the last, partial tile takes the general path."""
    lib = bq._lib.load()
    n, r = 24, (1 << 21) + 77
    streams = [markov(lib, 5, i, r, 40.0, 60000.0) for i in range(n)]
    acc = [(k == 0 or k >= 3) if acc_kind == "zero_accepted" else (k in (2, 5)) for k in range(n + 1)]
    q = bq.RleQuery(dev(streams), r)
    nw = (r + 63) // 64
    for _ in range(2):  # per-stream path, then the sliced layout
        out, pc = q.symmetric(acc)
        exp = O.cdom_symmetric(streams, r, acc)
        assert np.array_equal(host(out, nw), exp)
        assert int(pc.item()) == popcount(exp)


def test_concurrent_evaluations_share_one_query(bq, monkeypatch):
    """Several host threads evaluate one query (the reference allows concurrent
    invocations on shared inputs); the layout is built once and
    every answer matches the oracle."""
    import threading

    monkeypatch.delenv("BQ_RLE_SLICED", raising=False)
    lib = bq._lib.load()
    n, r = 64, 1 << 20
    streams = [markov(lib, 31, i, r, 64.0, 700.0) for i in range(n)]
    q = bq.RleQuery(dev(streams), r)
    nw = r // 64
    ts = [1, 3, 7, 20, 64]
    exp = {t: O.cdom_threshold(streams, r, t) for t in ts}
    errors = []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    t = ts[(k + rep) % len(ts)]
                    out, pc = q.threshold(t)
                    s.synchronize()
                    if not np.array_equal(host(out, nw), exp[t]):
                        errors.append((k, t))
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors
    assert q.layout_stats[0] > 0


@pytest.mark.parametrize("world", [2, 3, 7])
def test_word_range_queries_tile_the_result(bq, world):
    """Replicated streams, one query per 1024-aligned word range (the multi-GPU RLE
    shard, here all on one GPU): the windows concatenate to the
    whole result and their popcounts add up; both evaluations (K4, then K4s)."""
    from paper_1402_4073_b200.shard import shard_range

    lib = bq._lib.load()
    n, r = 50, 64 * 9000 - 11
    nw = (r + 63) // 64
    streams = [markov(lib, 13, i, r, 48.0, 500.0) for i in range(n)]
    d = dev(streams)
    qs = [bq.RleQuery(d, r, word_range=shard_range(nw, world, g, 1024)) for g in range(world)]
    for t in (1, 4, 9):
        exp = O.cdom_threshold(streams, r, t)
        for _ in range(2):
            parts, total = [], 0
            for q in qs:
                b, e = q.word_range
                out, pc = q.threshold(t)
                parts.append(host(out, e - b) if e > b else np.zeros(0, dtype=np.uint64))
                total += int(pc.item())
            assert np.array_equal(np.concatenate(parts), exp), t
            assert total == popcount(exp)


def test_word_range_errors(bq):
    lib = bq._lib.load()
    r = 64 * 5000
    d = dev([markov(lib, 1, 0, r, 8.0, 100.0)])
    with pytest.raises(bq.InputError):
        bq.RleQuery(d, r, word_range=(512, 2048))  # not tile aligned
    with pytest.raises(bq.InputError):
        bq.RleQuery(d, r, word_range=(1024, 1500))  # interior end not aligned
    q = bq.RleQuery(d, r, word_range=(4096, 10 ** 9))  # end clamps to ceil(r/64)
    assert q.word_range == (4096, 5000)


def test_max_inputs_rle(bq):
    """N = BQ_MAX_INPUTS (65535) RLE streams: the directory's per-stream grid
    dimension at its limit and 16-bit packed counts reaching N (all-ones words)."""
    lib = bq._lib.load()
    n, r = 65535, 64 * 1500 + 7
    nw = (r + 63) // 64
    rng = np.random.default_rng(65535)
    ones = np.full(nw, 2**64 - 1, dtype=np.uint64)
    ones[-1] = np.uint64((1 << 7) - 1)
    pool = [O.rle_compress(ones, r), np.zeros(0, dtype=np.uint64)]
    for k in range(6):
        w = np.zeros(nw, dtype=np.uint64)
        idx = rng.integers(0, nw, size=40)
        w[idx] = rng.integers(1, 2**63, size=40, dtype=np.uint64)
        w[-1] &= np.uint64((1 << 7) - 1)
        pool.append(O.rle_compress(O.trim(w), r))
    streams = [pool[0] if i % 3 == 0 else pool[1 + i % (len(pool) - 1)] for i in range(n)]
    flat = np.concatenate([s for s in streams if s.size] + [np.zeros(1, dtype=np.uint64)])
    dflat = torch.from_numpy(flat.view(np.int64)).cuda()
    d, o = [], 0
    for s in streams:
        d.append(bq.DeviceRleBitmap(dflat[o:o + s.size] if s.size else dflat[:0], r, s.size))
        o += s.size
    q = bq.RleQuery(d, r)
    for t in (1, n // 3, n // 3 + 1, n):
        for _ in range(2):  # K4, then K4s
            out, pc = q.threshold(t)
            exp = O.cdom_threshold(streams, r, t)
            assert np.array_equal(host(out, nw), exp), t
            assert int(pc.item()) == popcount(exp)


def test_release_cached_memory_between_queries(bq):
    """Queries take their directory and layout from libbq's memory pool; returning
    the cached memory to the driver between queries leaves later queries correct."""
    lib = bq._lib.load()
    n, r = 40, 1 << 19
    streams = [markov(lib, 9, i, r, 64.0, 2000.0) for i in range(n)]
    nw = r // 64
    for _ in range(2):
        q = bq.RleQuery(dev(streams), r)
        for t in (2, 5):
            out, pc = q.threshold(t)
            exp = O.cdom_threshold(streams, r, t)
            assert np.array_equal(host(out, nw), exp), t
        q.close()
        bq.release_cached_memory()


@pytest.mark.parametrize("chunk", ["1", "3", "4"])
def test_first_evaluation_in_chunks(bq, chunk, monkeypatch):
    """K4 + K4c launched over chunks of tiles (BQ_K4_CHUNK; by default 65536 tiles bound
    the deferred-count scratch): every chunk's deferred tiles are resolved, on the whole
    range and on a word-range query, at thresholds where most tiles reach phase C."""
    monkeypatch.setenv("BQ_K4_CHUNK", chunk)
    lib = bq._lib.load()
    n, r = 40, 64 * 9000 - 5
    nw = (r + 63) // 64
    streams = [markov(lib, 29, i, r, 48.0, 400.0) for i in range(n)]
    d = dev(streams)
    for t in (2, 5, 11):
        exp = O.cdom_threshold(streams, r, t)
        q = bq.RleQuery(d, r)
        out, pc = q.threshold(t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
        q.close()
        q = bq.RleQuery(d, r, word_range=(2048, 7168))
        out, pc = q.threshold(t)
        assert np.array_equal(host(out, 5120), exp[2048:7168]), t
        q.close()
