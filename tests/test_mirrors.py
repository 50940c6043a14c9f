"""The package's own bitmap types (bitmaps.py) mirror the reference API
(bitmaps.py:54-345) so the package is a drop-in without the reference
installed: run lists, word segments, cardinality, membership, positions and
run counts agree with the reference's on random bitmaps.  CPU only (the
operators &, |, ^, andnot run on the device and are covered by the GPU tests)."""

from __future__ import annotations

import os
import random
import sys

import pytest

from paper_1402_4073_b200 import bitmaps as M
from paper_1402_4073_b200.errors import FormatError, InputError

REF = os.environ.get("BQ_REFERENCE_SRC", "/root/reference/pkg/src")


def _words(rng, r, kind):
    nw = (r + 63) // 64
    out = []
    for _ in range(nw):
        if kind == "zero":
            w = 0
        elif kind == "one":
            w = (1 << 64) - 1
        elif kind == "sparse":
            w = rng.getrandbits(64) & rng.getrandbits(64) & rng.getrandbits(64)
        elif kind == "dense":
            w = rng.getrandbits(64) | rng.getrandbits(64)
        else:
            w = rng.choice([0, (1 << 64) - 1, rng.getrandbits(64)])
        out.append(w)
    if r % 64 and nw:
        out[-1] &= (1 << (r % 64)) - 1
    return out


def test_mirrors_without_reference():
    u = M.UncompressedBitmap.from_positions([1, 2, 7, 9], 16)
    assert u.words == [0b1010000110] and list(u.iter_runs()) == [(0, 0, 0), (1, 2, 1), (3, 6, 0), (7, 7, 1),
                                                                 (8, 8, 0), (9, 9, 1), (10, 15, 0)]
    mk = lambda bit, run, dirty: bit | (run << 1) | (dirty << 33)  # noqa: E731
    r = M.RleBitmap([mk(1, 2, 1), 0x5], 64 * 10)  # implicit zero tail
    assert list(r.iter_word_segments()) == [("f", 1, 2), ("d", 1, 1), ("f", 0, 7)]
    assert r.cardinality() == 130 and r.get(128) and not r.get(129) and r.get(130)
    assert r.positions()[-2:] == [128, 130] and r.run_count() == 4
    with pytest.raises(FormatError):
        list(M.RleBitmap([mk(0, 1, 3), 1], 640).iter_word_segments())
    with pytest.raises(FormatError):
        list(M.RleBitmap([mk(0, 11, 0)], 640).iter_word_segments())
    with pytest.raises(InputError):
        r.get(640)
    assert list(M.UncompressedBitmap.empty(0).iter_runs()) == []


def test_mirrors_match_the_reference():
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    sys.path.insert(0, REF)
    from bitquorum import bitmaps as R

    rng = random.Random(1)
    for _ in range(150):
        r = rng.choice([0, 1, 63, 64, 65, 200, 1000, 3000])
        kind = rng.choice(["runs", "sparse", "dense", "zero", "one"])
        words = _words(rng, r, kind)
        ru, mu = R.UncompressedBitmap(list(words), r), M.UncompressedBitmap(list(words), r)
        assert list(ru.iter_runs()) == list(mu.iter_runs())
        assert ru.positions() == mu.positions() and ru.cardinality() == mu.cardinality()
        rc = R.compress(ru)
        mc = M.RleBitmap(list(rc.words), r)
        assert list(rc.iter_word_segments()) == list(mc.iter_word_segments())
        assert list(rc.iter_word_segments(rc.bit_length // 64 + 3)) == list(mc.iter_word_segments(r // 64 + 3))
        assert rc.cardinality() == mc.cardinality() and rc.positions() == mc.positions()
        assert list(rc.iter_runs()) == list(mc.iter_runs()) and rc.run_count() == mc.run_count()
        for p in range(0, r, max(1, r // 17)):
            assert rc.get(p) == mc.get(p) and ru.get(p) == mu.get(p)
        assert M.RleBitmap.empty(r).words == R.RleBitmap.empty(r).words
