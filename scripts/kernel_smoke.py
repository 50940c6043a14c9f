"""Exercise every libbq kernel family on small inputs (run with BQ_RLE_SLICED=1
and =0 for both RLE paths, K4s and K4):
K1/K2 (all epilogues, ragged inputs, word ranges), K3/K4/K4s (phase C
included), the device encoder, set algebra, the program JIT, the host
streaming path and the membership kernels.  Exits 0 when every result matches
the CPU oracle."""

from __future__ import annotations

import ctypes
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1402_4073_b200 as bq  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1402_4073_b200 import _lib  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def main():
    lib = _lib.load()
    rng = np.random.default_rng(0)
    n, r = 37, 64 * 700 + 5
    nw = (r + 63) // 64
    arrs = []
    for i in range(n):
        a = rng.integers(0, 2**64 - 1, size=nw, dtype=np.uint64, endpoint=True) & \
            rng.integers(0, 2**64 - 1, size=nw, dtype=np.uint64, endpoint=True)
        a[-1] &= np.uint64((1 << 5) - 1)
        arrs.append(a[: nw - (i * 13) % 200])
    q = bq.ThresholdQuery([dev(a) for a in arrs], r)
    for t in (1, 2, 9, n):
        out, _ = q.threshold(t)
        assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), O.scan_count(arrs, r, t)), t
    for acc in ([2 <= k <= 9 for k in range(n + 1)], [bool(rng.random() < .5) for _ in range(n + 1)],
                [k % 2 == 1 for k in range(n + 1)]):
        out, _ = q.symmetric(acc)
        assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), O.scan_count_symmetric(arrs, r, acc))
    qr = bq.ThresholdQuery([dev(a) for a in arrs], r, word_range=(512, nw))
    out, _ = qr.threshold(5)
    assert np.array_equal(out[: nw - 512].cpu().numpy().view(np.uint64), O.scan_count(arrs, r, 5)[512:])
    outs, _ = bq.sweep_host(arrs, r, [3, [k == 2 for k in range(n + 1)]], chunk_words=1024)
    assert np.array_equal(outs[0], O.scan_count(arrs, r, 3))

    # RLE: staged and unstaged phase A, phase C, malformed input
    streams = []
    for i in range(n):
        cap = 4 * nw + 64
        buf = np.empty(cap, dtype=np.uint64)
        k = ctypes.c_uint64(0)
        assert lib.bq_gen_markov_rle(5, i, r, 40.0, 200.0, buf.ctypes.data, cap, ctypes.byref(k)) == 0
        streams.append(buf[: k.value].copy())
    for _ in range(1):
        rq = bq.RleQuery([bq.DeviceRleBitmap(dev(s), r) for s in streams], r)
        for t in (1, 3, n):
            out, _ = rq.threshold(t)
            assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), O.cdom_threshold(streams, r, t)), t
        acc = [k % 3 == 1 for k in range(n + 1)]
        out, _ = rq.symmetric(acc)
        assert np.array_equal(out[:nw].cpu().numpy().view(np.uint64), O.cdom_symmetric(streams, r, acc))
    try:
        bq.RleQuery([bq.DeviceRleBitmap(dev(np.array([(3 << 33)], dtype=np.uint64)), 640)], 640)
        raise AssertionError("malformed stream accepted")
    except bq.FormatError:
        pass

    # encoder, set algebra, program JIT, membership
    from paper_1402_4073_b200.api import compress_words, encode_device
    w = arrs[0]
    assert encode_device(dev(w), r).tolist() == compress_words(w, r)
    a = bq.UncompressedBitmap(arrs[1].tolist(), r)
    b = bq.UncompressedBitmap(arrs[2].tolist(), r)
    got = bq.binary_op("xor", a, b)
    x = np.zeros(nw, dtype=np.uint64)
    x[: arrs[1].size] ^= arrs[1]
    x[: arrs[2].size] ^= arrs[2]
    assert np.array_equal(np.array(got.words + [0] * (nw - len(got.words)), dtype=np.uint64), x)
    prog = types.SimpleNamespace(arity=3, n_slots=5, result_slot=4,
                                 instructions=[(2, 3, 0, 1), (4, 4, 3, 2), (7, 3, -1, -1)])
    ins3 = [bq.UncompressedBitmap(arrs[k].tolist(), r) for k in range(3)]
    got = bq.execute(prog, ins3)
    y = np.zeros(nw, dtype=np.uint64)
    p0, p1, p2 = (np.pad(arrs[k], (0, nw - arrs[k].size)) for k in range(3))
    y = (p0 & p1) ^ p2
    assert np.array_equal(np.array(got.words + [0] * (nw - len(got.words)), dtype=np.uint64), y)
    from paper_1402_4073_b200.similarity import membership
    m = membership(ins3, [0, 77, 64 * 300 + 3])
    assert m.shape == (3, 3)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
