"""Error contract and resource hygiene of the device path: caller-supplied result
buffers are validated (no out-of-bounds or misaligned 128-bit stores), bit_length-0
RLE streams are still validated as the reference's iter_word_segments does
(bitmaps.py:196-219), cached LUT tables give stable results, destroys do not
change the caller's current device, and the query cache respects the upload
cache's byte bound.  Needs a B200."""

from __future__ import annotations

import gc

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


def _rle_query(bq, streams, r):
    ts = [torch.from_numpy(np.ascontiguousarray(s, dtype=np.uint64).view(np.int64)).cuda() for s in streams]
    return bq.RleQuery([bq.DeviceRleBitmap(t, r, t.numel()) for t in ts], r), ts


def _markov(n, r):
    return [O.gen_markov_rle(7, i, r, 96.0, 900.0) for i in range(n)]


def test_rle_out_buffer_is_validated(bq):
    r = 1 << 16
    q, _keep = _rle_query(bq, _markov(4, r), r)
    nw = q.out_words
    buf = torch.zeros(nw + 2, dtype=torch.int64, device="cuda")
    with pytest.raises(bq.InputError):
        q.threshold(2, out=buf[: nw - 1])  # too short
    with pytest.raises(bq.InputError):
        q.threshold(2, out=buf[1 : nw + 1])  # 8-byte aligned only
    with pytest.raises(bq.InputError):
        q.threshold(2, out=torch.zeros(nw, dtype=torch.int32, device="cuda"))
    out, pc = q.threshold(2, out=buf[2 : nw + 2])  # 16-byte aligned view: accepted
    torch.cuda.synchronize()
    exp = O.cdom_threshold(_markov(4, r), r, 2)
    assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp)
    q.close()


def test_c_abi_rejects_misaligned_rle_output(bq):
    import ctypes

    lib = bq._lib.load()
    r = 1 << 12
    q, _keep = _rle_query(bq, _markov(2, r), r)
    buf = torch.zeros(q.out_words + 2, dtype=torch.int64, device="cuda")
    rc = lib.bq_rle_query_threshold(q._h, 1, ctypes.c_void_p(buf.data_ptr() + 8), None, None)
    assert rc == -1 and b"aligned" in lib.bq_last_error()
    q.close()


@pytest.mark.parametrize("words,ok", [
    ([], True), ([0], True), ([1, 0, 1], True),           # empty markers only
    ([0x2], False),                                      # a fill of one word: beyond bit_length 0
    ([1 << 33, 5], False),                               # one literal word
    ([1 << 33], False),                                  # truncated literal group
    ([0x2, 2 << 33, 5], False),                          # overlong, then truncated: FormatError either way
])
def test_rle_bit_length_zero_streams_are_validated(bq, words, ok):
    s = np.asarray(words, dtype=np.uint64)
    t = torch.from_numpy(s.view(np.int64)).cuda() if s.size else torch.zeros(1, dtype=torch.int64, device="cuda")
    d = bq.DeviceRleBitmap(t, 0, s.size)
    if ok:
        q = bq.RleQuery([d], 0)
        assert q.out_words == 0
        q.close()
    else:
        with pytest.raises(bq.FormatError):
            bq.RleQuery([d], 0)


def test_lut_symmetric_spec_cached_and_stable(bq):
    """A MODE_LUT spec (many accept[] changes) evaluated repeatedly and alternated
    with another: identical words and popcounts each time (the per-query table cache)."""
    n, nw = 40, 4096
    rng = np.random.default_rng(5)
    host = [rng.integers(0, 2**63, nw, dtype=np.uint64) & rng.integers(0, 2**63, nw, dtype=np.uint64)
            for _ in range(n)]
    dev = [torch.from_numpy(a.view(np.int64)).cuda() for a in host]
    q = bq.ThresholdQuery(dev, 64 * nw)
    specs = [[bool((k * 7 + 3) % 5 < 2) for k in range(n + 1)], [bool(k % 3 == 1) for k in range(n + 1)]]
    exp = [O.scan_count_symmetric(host, 64 * nw, s) for s in specs]
    for rep in range(6):
        k = rep % 2
        out, pc = q.symmetric(specs[k])
        torch.cuda.synchronize()
        got = out[:nw].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, exp[k])
        assert int(pc.item()) == int(np.unpackbits(exp[k].view(np.uint8)).sum())
    q.close()


def test_destroy_keeps_the_current_device(bq):
    torch.cuda.set_device(0)
    r = 1 << 14
    q, _keep = _rle_query(bq, _markov(3, r), r)
    q.threshold(2)
    q2 = bq.ThresholdQuery([torch.zeros(r // 64, dtype=torch.int64, device="cuda")], r, device=0)
    q2.threshold(1)
    del q, q2
    gc.collect()
    torch.cuda.synchronize()
    assert torch.cuda.current_device() == 0


def test_query_cache_respects_upload_byte_bound(bq):
    from paper_1402_4073_b200 import api
    from paper_1402_4073_b200.bitmaps import UncompressedBitmap

    nw = 1 << 14
    cache = api._QueryCache(maxsize=32, max_bytes=3 * 8 * nw * 4)  # room for ~3 four-input queries
    rng = np.random.default_rng(11)
    dev = torch.device("cuda", 0)
    for k in range(8):
        bms = [UncompressedBitmap(rng.integers(1, 2**63, nw, dtype=np.uint64).tolist(), 64 * nw) for _ in range(4)]
        cache.get("u", bms, 64 * nw, dev)
        assert cache.held_bytes <= cache.max_bytes or len(cache._d) == 1
    assert len(cache._d) <= 3
    cache.clear()
