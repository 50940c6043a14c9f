"""Parity of the CUDA counting kernels (K1/K2) with the reference, through the
C ABI (ctypes) and the drop-in Python entry points.  Needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, load_kat, padded
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

THRESH = load_golden("threshold")
SYM = load_golden("symmetric")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def dev(arrs):
    return [torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda() for a in arrs]


def host(t, nw):
    return t[:nw].cpu().numpy().view(np.uint64)


def popcount(words):
    return int(np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8)).sum())


def gen(lib, seed, i, q, nw):
    a = np.empty(nw, dtype=np.uint64)
    assert lib.bq_gen_bernoulli(seed, i, q, 0, nw, a.ctypes.data, 0, None) == 0
    return a


# ---------------------------------------------------------------------------
# golden cases produced by the reference (tests/golden/make_golden.py)

@pytest.mark.parametrize("case", THRESH, ids=lambda c: c.id)
def test_threshold_golden_capi(bq, case):
    q = bq.ThresholdQuery(dev(case.inputs), case.r)
    out, pc = q.threshold(case.meta["t"])
    nw = (case.r + 63) // 64
    assert np.array_equal(host(out, nw), padded(case.out, case.r))
    assert int(pc.item()) == case.meta["card"]


@pytest.mark.parametrize("case", THRESH[::3], ids=lambda c: c.id)
def test_threshold_golden_dropin(bq, case):
    """Reference-style host bitmaps in, reference-style (trimmed) words out."""
    ins = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    t = case.meta["t"]
    stats = {}
    got = bq.scan_count(ins, t, stats=stats)
    assert isinstance(got, bq.UncompressedBitmap)
    assert got.words == case.out.tolist()
    assert got.bit_length == case.r
    assert got.cardinality() == case.meta["card"]
    assert stats["counter_width"] == bq.counter_width(len(ins))
    assert bq.looped_threshold(ins, t).words == case.out.tolist()
    if 2 <= t < len(ins):
        assert bq.csv_threshold(ins, t).words == case.out.tolist()


@pytest.mark.parametrize("case", SYM, ids=lambda c: c.id)
def test_symmetric_golden(bq, case):
    q = bq.ThresholdQuery(dev(case.inputs), case.r)
    out, pc = q.symmetric(case.meta["accept"])
    nw = (case.r + 63) // 64
    assert np.array_equal(host(out, nw), padded(case.out, case.r))
    assert int(pc.item()) == case.meta["card"]
    ins = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    assert bq.scan_count_symmetric(ins, bq.SymmetricSpec(tuple(bool(a) for a in case.meta["accept"]))).words \
        == case.out.tolist()


def test_generator_device_matches_pin(bq):
    kat = load_kat()["generator"]
    lib = bq._lib.load()
    for c in kat["cases"]:
        d = torch.empty(2, dtype=torch.int64, device="cuda")
        assert lib.bq_gen_bernoulli(kat["seed"], c["bitmap"], c["q"], c["word"], 1, d.data_ptr(), 1,
                                    torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        assert int(host(d, 1)[0]) == int(c["value"])


# ---------------------------------------------------------------------------
# random cases against the oracle, covering every epilogue and counter width

@pytest.mark.parametrize("n", [1, 2, 3, 7, 15, 16, 17, 31, 33, 64, 100, 255, 256, 511, 1024, 4100])
def test_threshold_random_all_t(bq, n):
    lib = bq._lib.load()
    rng = np.random.default_rng(n)
    r = int(rng.integers(1, 3000)) * 64 - int(rng.integers(0, 64))
    nw = (r + 63) // 64
    arrs = []
    for i in range(n):
        q = int(rng.choice([0, 300, 6554, 32768, 60000, 65536]))
        a = gen(lib, 7, i, q, nw)
        a[-1] &= np.uint64((1 << (r % 64)) - 1) if r % 64 else np.uint64(2**64 - 1)
        cut = nw if rng.random() < 0.7 else int(rng.integers(0, nw + 1))  # ragged trimmed inputs
        arrs.append(a[:cut])
    qry = bq.ThresholdQuery(dev(arrs), r)
    ts = sorted({1, 2, 3, n, max(1, n // 2), max(1, n - 1), int(rng.integers(1, n + 1))} & set(range(1, n + 1)))
    for t in ts:
        out, pc = qry.threshold(t)
        exp = O.threshold_port(arrs, r, t)
        got = host(out, nw)
        assert np.array_equal(got, exp), f"n={n} t={t}"
        assert int(pc.item()) == popcount(exp)


@pytest.mark.parametrize("n,spec", [(5, "parity"), (64, "parity"), (100, "mod4"), (300, "many"),
                                    (40, "const1"), (40, "const0"), (256, "interval"), (1000, "many"),
                                    (9, "delta0")])
def test_symmetric_modes(bq, n, spec):
    lib = bq._lib.load()
    rng = np.random.default_rng(1000 + n)
    r = 64 * 700 + 13
    nw = (r + 63) // 64
    arrs = [gen(lib, 11, i, int(rng.choice([3277, 32768, 50000])), nw) for i in range(n)]
    for a in arrs:
        a[-1] &= np.uint64((1 << 13) - 1)
    if spec == "parity":
        acc = [k % 2 == 1 for k in range(n + 1)]
    elif spec == "mod4":
        acc = [k % 4 in (1, 2) for k in range(n + 1)]
    elif spec == "many":
        acc = [bool(rng.random() < 0.5) for _ in range(n + 1)]
    elif spec == "const1":
        acc = [True] * (n + 1)
    elif spec == "const0":
        acc = [False] * (n + 1)
    elif spec == "delta0":
        acc = [k == 0 for k in range(n + 1)]
    else:
        acc = [2 <= k <= 10 for k in range(n + 1)]
    qry = bq.ThresholdQuery(dev(arrs), r)
    out, pc = qry.symmetric(acc)
    exp = O.symmetric_port(arrs, r, acc)
    assert np.array_equal(host(out, nw), exp)
    assert int(pc.item()) == popcount(exp)


def test_word_range_shards_tile_the_result(bq):
    from paper_1402_4073_b200.shard import shard_range

    lib = bq._lib.load()
    n, r = 37, 64 * 5000 - 9
    nw = (r + 63) // 64
    arrs = [gen(lib, 3, i, 6554 * (1 + i % 5), nw - (i * 37) % 900) for i in range(n)]
    for a in arrs:
        if a.size == nw:
            a[-1] &= np.uint64((1 << 55) - 1)
    full = bq.ThresholdQuery(dev(arrs), r)
    out, pc = full.threshold(9)
    whole = host(out, nw)
    d = dev(arrs)
    total_pc = 0
    for world in (2, 3, 8):
        parts = []
        total_pc = 0
        for g in range(world):
            b, e = shard_range(nw, world, g)
            q = bq.ThresholdQuery(d, r, word_range=(b, e))
            o, p = q.threshold(9)
            parts.append(host(o, e - b))
            total_pc += int(p.item())
        assert np.array_equal(np.concatenate(parts), whole)
        assert total_pc == int(pc.item())


def test_sweep_host_matches_device(bq):
    lib = bq._lib.load()
    n, r = 64, 64 * 20000 + 1
    nw = (r + 63) // 64
    arrs = [gen(lib, 5, i, 655 + 500 * i, nw) for i in range(n)]
    for a in arrs:
        a[-1] &= np.uint64(1)
    arrs[3] = arrs[3][: nw // 2]
    queries = [1, 2, 16, 32, 64, [2 <= k <= 10 for k in range(n + 1)]]
    outs, pcs = bq.sweep_host(arrs, r, queries, chunk_words=4096)
    q = bq.ThresholdQuery(dev(arrs), r)
    for k, qq in enumerate(queries):
        o, p = q.threshold(qq) if isinstance(qq, int) else q.symmetric(qq)
        assert np.array_equal(outs[k], host(o, nw)), k
        assert pcs[k] == int(p.item())


def test_c1_full_size(bq):
    """Config 1 at full size: N=8, r=2^20, p=0.1 (q=6554), T=3, output + popcount."""
    lib = bq._lib.load()
    n, r, nw = 8, 1 << 20, 1 << 14
    arrs = [gen(lib, 1402, i, 6554, nw) for i in range(n)]
    q = bq.ThresholdQuery(dev(arrs), r)
    out, pc = q.threshold(3)
    exp = O.scan_count(arrs, r, 3)
    assert np.array_equal(host(out, nw), exp)
    assert int(pc.item()) == popcount(exp)


def test_errors(bq):
    lib = bq._lib.load()
    arrs = [gen(lib, 1, i, 32768, 64) for i in range(4)]
    q = bq.ThresholdQuery(dev(arrs), 64 * 64)
    with pytest.raises(bq.InputError):
        q.threshold(0)
    with pytest.raises(bq.InputError):
        q.threshold(5)
    with pytest.raises(bq.InputError):
        q.symmetric([True] * 4)  # arity mismatch
    with pytest.raises(bq.InputError):
        bq.ThresholdQuery(dev(arrs), 64 * 63)  # more words than bit_length allows
    with pytest.raises(bq.InputError):
        bq.scan_count([bq.UncompressedBitmap([1], 64), bq.RleBitmap([], 64)], 1)  # mixed representations
    with pytest.raises(bq.ResourceError):
        bq.scan_count([bq.UncompressedBitmap([1], 1 << 40)], 1, budget_bytes=1 << 20)


@pytest.mark.parametrize("n", [8200, 20000, 65535])
def test_large_n_global_pointer_table(bq, n):
    """N > 8192: the kernel reads the pointer table from global memory; M = 14/16-bit counters."""
    lib = bq._lib.load()
    nw = 96
    r = 64 * nw - 3
    arrs = []
    for i in range(n):
        a = gen(lib, 21, i, 32768 if i % 3 else 65000, nw)
        a[-1] &= np.uint64((1 << 61) - 1)
        arrs.append(a[: nw - (i % 7)])
    q = bq.ThresholdQuery(dev(arrs), r)
    for t in (1, n // 2, n - 3, n):
        out, pc = q.threshold(t)
        exp = O.threshold_port(arrs, r, t)
        assert np.array_equal(host(out, nw), exp), t
        assert int(pc.item()) == popcount(exp)
    rng = np.random.default_rng(n)
    acc = [bool(rng.random() < 0.5) for _ in range(n + 1)]  # many breakpoints -> LUT epilogue
    out, pc = q.symmetric(acc)
    exp = O.scan_count_symmetric(arrs, r, acc)
    assert np.array_equal(host(out, nw), exp)
    assert int(pc.item()) == popcount(exp)
