"""Edge cases of the one-pass RLE directory (K3, csrc/bq_rle_dir.cu): the
speculative per-segment entry guesses and their repair, literal groups spanning
segments (32 words) and blocks (1024 words) and the decoupled look-back between
blocks, streams whose length is exactly a segment / block multiple, streams
shorter than the guess window, 8-byte-misaligned stream starts, adversarial
literal words that look like markers, and validation failures (truncated,
overlong, bits beyond r) placed in late blocks.  Each case is checked against
the oracle's decoder / cdom sweep (pinned to the reference).  Needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MASK = (1 << 64) - 1


def mk(bit, run, dirty):
    return bit | (run << 1) | (dirty << 33)


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def _query(bq, streams, r, misalign=False, range_=None):
    """Streams packed back to back in one buffer (8-byte-aligned starts when
    misalign), through RleQuery.from_packed."""
    pad = 1 if misalign else 0
    offs, lens, flat = [], [], [np.zeros(pad, dtype=np.uint64)]
    o = pad
    for s in streams:
        offs.append(o)
        lens.append(s.size)
        flat.append(s)
        o += s.size
    flat.append(np.zeros(2, dtype=np.uint64))
    buf = torch.from_numpy(np.concatenate(flat).view(np.int64)).cuda()
    q = bq.RleQuery.from_packed(buf, offs, lens, r, word_range=range_)
    return q, buf


def _rand_literal(rng, n):
    # literal words that are never fills; half of them look like markers with small dirty fields
    w = rng.integers(1, 2**63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    small = rng.random(n) < 0.5
    w[small] = (w[small] & np.uint64((1 << 33) - 1)) | (rng.integers(0, 4, int(small.sum()), dtype=np.uint64) << np.uint64(33))
    w[w == np.uint64(MASK)] = np.uint64(5)
    return w


def _stream(rng, nwords_target, max_lit, long_every=0):
    """A valid stream of about nwords_target words: random fills and literal groups
    (occasionally max_lit long), plus its bit length."""
    out, covered = [], 0
    while len(out) < nwords_target:
        run = int(rng.integers(0, 40))
        lit = int(rng.integers(0, 4))
        if long_every and rng.random() < 1.0 / long_every:
            lit = int(rng.integers(max_lit // 2, max_lit + 1))
        bit = int(rng.integers(0, 2))
        out.append(mk(bit, run, lit))
        out.extend(int(x) for x in _rand_literal(rng, lit))
        covered += run + lit
    s = np.asarray(out, dtype=np.uint64)
    return s, covered * 64


def _check_decode(bq, streams, r, **kw):
    q, _buf = _query(bq, streams, r, **kw)
    nw = (r + 63) // 64
    for t in (1, len(streams)) if len(streams) > 1 else (1,):
        out, pc = q.threshold(t)
        exp = O.cdom_threshold(streams, r, t)
        got = out[: q.out_words].cpu().numpy().view(np.uint64)
        w0 = q.word_range[0]
        assert np.array_equal(got, exp[w0:w0 + q.out_words]), t
    q.close()
    return nw


@pytest.mark.parametrize("seed", range(6))
def test_long_literal_groups_cross_segments_and_blocks(bq, seed):
    """Literal groups of up to 5000 words: entries beyond a segment's first words,
    whole segments and blocks with no marker start (pass-through)."""
    rng = np.random.default_rng(seed)
    streams = []
    rmax = 0
    for i in range(5):
        s, r = _stream(rng, 20000, 5000, long_every=20)
        streams.append(s)
        rmax = max(rmax, r)
    _check_decode(bq, streams, rmax)


@pytest.mark.parametrize("length", [1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 127, 128, 129, 1023, 1024, 1025, 2047,
                                    2048, 2049, 3072, 3073, 4096, 4097])
def test_stream_lengths_at_segment_and_block_edges(bq, length):
    """Streams of exactly `length` words: one made of markers only (non-canonical
    adjacent fills, which the decoder must accept), one a single marker followed
    by length - 1 literal words (every later segment and block is inside it)."""
    rng = np.random.default_rng(length)
    markers = np.asarray([mk(0, 3, 0)] * (length - 1) + [mk(1, 2, 0)], dtype=np.uint64)
    literal = np.concatenate([np.asarray([mk(1, 1, length - 1)], dtype=np.uint64),
                              _rand_literal(rng, length - 1)]).astype(np.uint64)
    r = 64 * max(3 * (length - 1) + 2, length)
    _check_decode(bq, [markers, literal], r)


def test_misaligned_stream_starts(bq):
    rng = np.random.default_rng(11)
    streams, rmax = [], 0
    for _ in range(9):
        s, r = _stream(rng, int(rng.integers(1, 9000)), 300, long_every=50)
        streams.append(s)
        rmax = max(rmax, r)
    _check_decode(bq, streams, rmax, misalign=True)


def test_adversarial_literals_force_guess_repairs(bq):
    """Markers followed by literal words whose dirty fields are small: many
    speculative entries are wrong and must be repaired; the result stays exact."""
    rng = np.random.default_rng(5)
    out, covered = [], 0
    while len(out) < 50000:
        lit = int(rng.integers(1, 6))
        out.append(mk(int(rng.integers(0, 2)), int(rng.integers(0, 3)), lit))
        lw = rng.integers(1, 2**33, lit, dtype=np.uint64) | (rng.integers(0, 3, lit, dtype=np.uint64) << np.uint64(33))
        out.extend(int(x) for x in lw)
        covered += (out[-lit - 1] >> 1 & 0xFFFFFFFF) + lit
    s = np.asarray(out, dtype=np.uint64)
    r = 64 * covered
    _check_decode(bq, [s, s], r)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_validation_errors_in_late_blocks(bq, seed):
    rng = np.random.default_rng(seed)
    s, r = _stream(rng, 30000, 50)
    good = [s, s]
    _check_decode(bq, good, r)
    # truncated literal group at the end: the last marker with literals loses its last literal
    i, last = 0, None
    while i < s.size:  # follow the marker chain
        d = int(s[i]) >> 33
        if d:
            last = i
        i += 1 + d
    assert last is not None
    bad = s[: last + (int(s[last]) >> 33)]
    with pytest.raises(bq.FormatError):
        _query(bq, [s, bad], r)
    # overlong: a bit length one word short of the coverage
    with pytest.raises(bq.FormatError):
        _query(bq, [s], r - 64)
    # bits >= r: a one fill reaching the last (partial) word
    pref = O.rle_decompress(s, r)
    words = pref.copy()
    words[-1] = np.uint64(MASK)
    bad2 = O.rle_compress(words, r)
    with pytest.raises(bq.FormatError):
        _query(bq, [bad2], r - 5)


def test_range_shards_of_the_directory(bq):
    rng = np.random.default_rng(3)
    streams, rmax = [], 0
    for _ in range(6):
        s, r = _stream(rng, 40000, 400, long_every=30)
        streams.append(s)
        rmax = max(rmax, r)
    nw = (rmax + 63) // 64
    exp = O.cdom_threshold(streams, rmax, 2)
    b = (nw // 3) // 1024 * 1024
    e = (2 * nw // 3) // 1024 * 1024
    q, _buf = _query(bq, streams, rmax, range_=(b, e))
    out, _ = q.threshold(2)
    assert np.array_equal(out[: e - b].cpu().numpy().view(np.uint64), exp[b:e])
    q.close()
