"""Property-based parity (hypothesis): random small instances -- ragged
lengths, r % 64 != 0, any N / T / accept vector, both representations -- must
match the CPU oracle bit for bit, through the drop-in API and the C ABI."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

SETTINGS = settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


@st.composite
def instances(draw):
    n = draw(st.integers(1, 70))
    r = draw(st.integers(1, 64 * 80))
    seed = draw(st.integers(0, 2**32 - 1))
    style = draw(st.sampled_from(["uniform", "sparse", "dense", "runs", "mixed"]))
    rng = np.random.default_rng(seed)
    nw = (r + 63) // 64
    arrs, bits = [], []
    for i in range(n):
        ri = r if (i == 0 or rng.random() < 0.6) else int(rng.integers(0, r + 1))
        wi = (ri + 63) // 64
        kind = style if style != "mixed" else rng.choice(["uniform", "sparse", "dense", "runs", "zero", "one"])
        if kind == "uniform":
            a = rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True)
        elif kind == "sparse":
            a = rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True) & \
                rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True) & \
                rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True)
        elif kind == "dense":
            a = rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True) | \
                rng.integers(0, 2**64 - 1, size=wi, dtype=np.uint64, endpoint=True)
        elif kind == "zero":
            a = np.zeros(wi, dtype=np.uint64)
        elif kind == "one":
            a = np.full(wi, 2**64 - 1, dtype=np.uint64)
        else:  # runs of whole words
            cls = rng.integers(0, 3, size=max(wi, 1))
            a = np.where(cls == 0, 0, np.where(cls == 1, np.uint64(2**64 - 1),
                                               rng.integers(1, 2**63, size=max(wi, 1), dtype=np.uint64)))
            a = np.repeat(a.astype(np.uint64), rng.integers(1, 9, size=a.size))[:wi]
        a = a.astype(np.uint64)
        if wi and ri % 64:
            a[-1] &= np.uint64((1 << (ri % 64)) - 1)
        nz = np.flatnonzero(a)
        arrs.append(a[: nz[-1] + 1 if nz.size else 0])  # trimmed, as the reference stores words
        bits.append(ri)
    t = draw(st.integers(1, n))
    accept = draw(st.lists(st.booleans(), min_size=n + 1, max_size=n + 1))
    return arrs, bits, max(bits), t, accept


def _padded(words, r):
    out = np.zeros((r + 63) // 64, dtype=np.uint64)
    out[: len(words)] = words
    return out


@SETTINGS
@given(instances())
def test_threshold_and_symmetric_uncompressed(bq, inst):
    arrs, bits, r, t, accept = inst
    ins = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(arrs, bits)]
    exp_t = O.scan_count(arrs, r, t)
    exp_s = O.scan_count_symmetric(arrs, r, accept)
    got_t = bq.scan_count(ins, t)
    got_s = bq.scan_count_symmetric(ins, bq.SymmetricSpec(tuple(accept)))
    assert np.array_equal(_padded(np.array(got_t.words, dtype=np.uint64), r), exp_t)
    assert np.array_equal(_padded(np.array(got_s.words, dtype=np.uint64), r), exp_s)
    assert got_t.bit_length == r and got_s.bit_length == r


@SETTINGS
@given(instances())
def test_threshold_and_symmetric_rle(bq, inst):
    arrs, bits, r, t, accept = inst
    comp = [O.rle_compress(a, b) for a, b in zip(arrs, bits)]
    ins = [bq.RleBitmap(c.tolist(), b) for c, b in zip(comp, bits)]
    got_t = bq.cdom_threshold(ins, t)
    got_s = bq.cdom_symmetric(ins, bq.SymmetricSpec(tuple(accept)))
    exp_t = O.cdom_threshold(comp, r, t)
    exp_s = O.cdom_symmetric(comp, r, accept)
    assert got_t.words == O.rle_compress(O.trim(exp_t), r).tolist()
    assert got_s.words == O.rle_compress(O.trim(exp_s), r).tolist()


@SETTINGS
@given(instances())
def test_rle_both_paths_device_query(bq, inst):
    """The same random instance through K4 (BQ_RLE_SLICED=0) and K4s (=1), device
    streams, threshold and symmetric."""
    import os

    arrs, bits, r, t, accept = inst
    comp = [O.rle_compress(a, b) for a, b in zip(arrs, bits)]
    dev = [torch.from_numpy(c.view(np.int64)).cuda() if c.size else torch.zeros(1, dtype=torch.int64, device="cuda")
           for c in comp]
    streams = [bq.DeviceRleBitmap(d, b, c.size) for d, b, c in zip(dev, bits, comp)]
    nw = (r + 63) // 64
    exp_t = O.cdom_threshold(comp, r, t)
    exp_s = O.cdom_symmetric(comp, r, accept)
    prev = os.environ.get("BQ_RLE_SLICED")
    try:
        for mode in ("0", "1"):
            os.environ["BQ_RLE_SLICED"] = mode
            q = bq.RleQuery(streams, r)
            out, pc = q.threshold(t)
            assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp_t), mode
            out, pc = q.symmetric(accept)
            assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp_s), mode
            q.close()
    finally:
        if prev is None:
            os.environ.pop("BQ_RLE_SLICED", None)
        else:
            os.environ["BQ_RLE_SLICED"] = prev
