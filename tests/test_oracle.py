"""Pin the CPU oracle against fixtures produced by running the reference itself
(tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import load_golden, load_kat, padded
from oracle import oracle as O

THRESH = load_golden("threshold")
SYM = load_golden("symmetric")
RLE = load_golden("rle")
CODEC = load_golden("codec")


@pytest.mark.parametrize("case", THRESH, ids=lambda c: c.id)
def test_scan_count_matches_reference(case):
    t = case.meta["t"]
    exp = padded(case.out, case.r)
    assert np.array_equal(O.scan_count(case.inputs, case.r, t), exp)
    assert np.array_equal(O.threshold_port(case.inputs, case.r, t, threads=2), exp)
    assert int(sum(int(w).bit_count() for w in case.out)) == case.meta["card"]


@pytest.mark.parametrize("case", SYM, ids=lambda c: c.id)
def test_symmetric_matches_reference(case):
    acc = case.meta["accept"]
    exp = padded(case.out, case.r)
    assert np.array_equal(O.scan_count_symmetric(case.inputs, case.r, acc), exp)
    assert np.array_equal(O.symmetric_port(case.inputs, case.r, acc, threads=2), exp)


@pytest.mark.parametrize("case", RLE, ids=lambda c: c.id)
def test_cdom_matches_reference(case):
    exp_u = padded(np.array(case.meta["uncompressed"], dtype=np.uint64), case.r)
    st = {}
    if case.meta["kind"] == "cdom_threshold":
        got = O.cdom_threshold(case.inputs, case.r, case.meta["t"], stats=st)
    else:
        got = O.cdom_symmetric(case.inputs, case.r, case.meta["accept"], stats=st)
    assert np.array_equal(got, exp_u)
    assert st == case.meta["stats"]  # segments, heap_pops, branches (runmerge.py:237-240)
    # the reference returns the canonical encoding of those words
    assert np.array_equal(O.rle_compress(O.trim(got), case.r), case.out)


@pytest.mark.parametrize("case", CODEC, ids=lambda c: c.id)
def test_codec_matches_reference(case):
    kind = case.meta["kind"]
    if kind == "compress":
        assert np.array_equal(O.rle_compress(case.inputs[0], case.r), case.out)
        assert np.array_equal(O.rle_decompress(case.out, case.r), padded(case.inputs[0], case.r))
    elif case.meta["status"] == "ok":
        assert np.array_equal(O.rle_decompress(case.inputs[0], case.r), padded(case.out, case.r))
    else:
        with pytest.raises(O.OracleError) as ei:
            O.rle_decompress(case.inputs[0], case.r)
        assert ei.value.code == O.EFORMAT


def test_known_answers():
    kat = load_kat()
    assert O.brute_threshold([[1, 2, 7], [2, 7, 9], [7]], 2) == kat["brute_threshold_spec160"] == [2, 7]
    ins = [O.words_from_positions(p, 16) for p in ([1], [1], [2])]
    assert O.positions_of(O.threshold_port(ins, 16, 2)) == kat["csv_spec542"] == [1]
    assert O.rle_compress(np.zeros(0, np.uint64), 128).tolist() == kat["compress_empty128"] == [4]
    assert O.words_from_positions([1, 2, 7, 9], 16).tolist() == kat["from_positions_1279"]
    words = np.array([0, 2**64 - 1, 3, 0, 0, 7], dtype=np.uint64)
    assert [str(w) for w in O.rle_compress(O.trim(words), 64 * 6).tolist()] == kat["canonical_example"]


def test_complement_identity():
    """theta(T, B) = NOT theta(N - T + 1, NOT B)."""
    rng = np.random.default_rng(7)
    n, r = 13, 64 * 50 - 3
    ins = [rng.integers(0, 2**63, size=50, dtype=np.uint64) * np.uint64(2) for _ in range(n)]
    mask = np.uint64((1 << (r % 64)) - 1)
    for a in ins:
        a[-1] &= mask
    neg = [~a for a in ins]
    for a in neg:
        a[-1] &= mask
    for t in range(1, n + 1):
        lhs = O.scan_count(ins, r, t)
        rhs = ~O.scan_count(neg, r, n - t + 1)
        rhs[-1] &= mask
        assert np.array_equal(lhs, rhs)


def test_oracle_generator_matches_pin():
    """The oracle's generator restatement (bench.py's CPU legs use it instead of
    libbq.so) reproduces the independent pure-Python KATs."""
    kat = load_kat()["generator"]
    for c in kat["cases"]:
        got = O.gen_bernoulli(kat["seed"], c["bitmap"], c["q"], c["word"], 1)
        assert int(got[0]) == int(c["value"])
    assert [O.gen_density_q16(kat["seed"], i, 655, 32768) for i in range(64)] == kat["density_q"]


def test_oracle_generator_matches_product_generator():
    """Same words as csrc/bq_gen.h (Bernoulli windows) and bq_gen_markov_rle (C4 streams)."""
    import ctypes

    from paper_1402_4073_b200 import _lib

    lib = _lib.load()
    for i in (0, 9, 63):
        q = lib.bq_gen_density_q16(1402, i, 655, 32768)
        a = np.empty(777, dtype=np.uint64)
        assert lib.bq_gen_bernoulli(1402, i, q, 99991, 777, a.ctypes.data, 0, None) == 0
        assert np.array_equal(a, O.gen_bernoulli(1402, i, q, 99991, 777))
    r = (1 << 21) + 37
    for i in (0, 3):
        cap = 1 << 16
        buf = np.empty(cap, dtype=np.uint64)
        n = ctypes.c_uint64(0)
        assert lib.bq_gen_markov_rle(1402, i, r, 256.0, 12544.0, buf.ctypes.data, cap, ctypes.byref(n)) == 0
        assert np.array_equal(buf[: n.value], O.gen_markov_rle(1402, i, r, 256.0, 12544.0))


# ---- BASELINE configs pinned to reference-run outputs (tests/golden/baseline.npz) ----

def _baseline():
    import json

    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "baseline.npz"))
    return z, json.loads(str(z["meta"]))


def test_oracle_matches_reference_on_baseline_windows():
    """The oracle on the exact seeded inputs of C1, C2, C3 and C5 windows reproduces
    the reference's own outputs (make_golden.py baseline_cases)."""
    z, meta = _baseline()
    for name, m in meta.items():
        if name.startswith("c4"):
            continue
        n, w0, nw = m["n"], m["w0"], m["nw"]
        q16 = m["q16"] if isinstance(m["q16"], list) else [m["q16"]] * n
        rows = [O.gen_bernoulli(1402, i, q16[i], w0, nw) for i in range(n)]
        if name.startswith("c3"):
            acc = [2 <= k <= 10 for k in range(n + 1)]
            got = O.scan_count_symmetric(rows, 64 * nw, acc)
        else:
            got = O.threshold_port(rows, 64 * nw, m["t"], threads=2)
        assert np.array_equal(got, z[name]), name
        assert int(np.unpackbits(got.view(np.uint8)).sum()) == m["card"], name


def test_oracle_cdom_matches_reference_on_c4_prefix():
    """C4's 1024 Markov streams over their first 2^20 bits: the oracle's cdom sweep
    equals the reference's cdom_threshold at T = 5, 10, 20, 50."""
    z, meta = _baseline()
    streams = [O.gen_markov_rle(1402, i, 1 << 20, 256.0, 12544.0) for i in range(1024)]
    for t in (5, 10, 20, 50):
        m = meta[f"c4_t{t}"]
        st = {}
        got = O.cdom_threshold(streams, m["r"], t, stats=st)
        assert np.array_equal(got, z[f"c4_t{t}"]), t
        assert st == m["stats"], t
