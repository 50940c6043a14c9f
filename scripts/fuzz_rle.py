"""Randomised differential test of the RLE path at multi-tile sizes (GPU box).

    python scripts/fuzz_rle.py [seconds] [first_seed] [eval|validate]

Random instances of 1-300 streams over up to 12 tiles -- canonical encodings of
Markov / dense / sparse / all-literal words and valid non-canonical streams (empty
markers, split fills, runs ending on tile boundaries, implicit tails) -- are
evaluated through K3 + K4 / K4c (first evaluation) and K3 + K4s (tile-sliced layout)
at random thresholds, accept vectors and word-range shards, and compared with the
oracle's cdom sweep word for word.  ``validate`` instead corrupts single streams
(truncation, bumped dirty / run fields, bits past r, extra markers, random words) and
checks that K3 and the oracle's decompress accept or reject the same streams.  Prints
one line per failure and a summary; exit code 1 on any mismatch.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
import paper_1402_4073_b200 as bq  # noqa: E402


def marker(bit, run, dirty):
    return (dirty << 33) | (run << 1) | bit


def noncanonical(rng, total):
    out, cov = [], 0
    target = total if rng.random() < 0.5 else int(total * rng.random())
    while cov < target:
        kind = rng.random()
        if kind < 0.1:
            out.append(marker(int(rng.integers(2)), 0, 0))
            continue
        room = target - cov
        run = int(min(room, rng.choice([0, 1, 2, 5, 40, 700, 3000]) if kind < 0.9 else room))
        dirty = int(min(room - run, rng.choice([0, 0, 1, 2, 3, 17, 90])))
        edge = 1024 - (cov + run) % 1024
        if kind < 0.25 and edge <= room - run:
            if rng.random() < 0.5:
                run, dirty = run + edge, 0
            elif edge <= 90:
                dirty = edge
        out.append(marker(int(rng.integers(2)), run, dirty))
        for _ in range(dirty):
            w = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(2))
            out.append(w if rng.random() < 0.8 else (1 << 64) - 1)
        cov += run + dirty
    return np.array(out, dtype=np.uint64)


def canonical(rng, r, nw, style):
    if style == "markov":
        m1, m0 = float(rng.choice([8, 64, 256, 2000])), float(rng.choice([64, 1000, 12544, 100000]))
        return O.gen_markov_rle(int(rng.integers(1 << 30)), int(rng.integers(1 << 20)), r, m1, m0)
    w = np.zeros(nw, dtype=np.uint64)
    if style == "literal":
        w = rng.integers(1, 2**63, size=nw, dtype=np.uint64)
    elif style == "sparse":
        idx = rng.integers(0, nw, size=max(1, nw // int(rng.choice([3, 20, 200]))))
        w[idx] = rng.integers(1, 2**63, size=idx.size, dtype=np.uint64)
    elif style == "windows":
        for _ in range(int(rng.integers(1, 8))):
            a = int(rng.integers(0, nw))
            b = min(nw, a + int(rng.choice([1, 30, 200, 1500])))
            w[a:b] = rng.integers(0, 2**64 - 1, size=b - a, dtype=np.uint64) if rng.random() < 0.6 else np.uint64(2**64 - 1)
    elif style == "short":
        k = int(rng.integers(0, nw + 1))
        w[:k] = rng.integers(0, 2**64 - 1, size=k, dtype=np.uint64)
    if r % 64:
        w[-1] &= np.uint64((1 << (r % 64)) - 1)
    return O.rle_compress(O.trim(w), r)


def run_case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 7, 31, 33, 64, 130, 300]))
    tiles = int(rng.choice([1, 2, 3, 4, 5, 8, 9, 12]))
    if rng.random() < 0.5:
        total = tiles * 1024 - int(rng.integers(0, 1024))
        r = 64 * total - int(rng.integers(0, 64))
    else:
        total = tiles * 1024
        r = 64 * total
    r = max(r, 1)
    nw = (r + 63) // 64
    noncanon = rng.random() < 0.4 and r % 64 == 0
    styles = ["markov", "literal", "sparse", "windows", "short"]
    streams = []
    for i in range(n):
        if noncanon:
            streams.append(noncanonical(rng, nw))
        else:
            st = styles[int(rng.integers(len(styles)))] if n > 31 or rng.random() < 0.7 else "markov"
            if st == "literal" and n * nw > 400000:
                st = "sparse"
            streams.append(canonical(rng, r, nw, st))
    dev = []
    for a in streams:
        t = torch.from_numpy(a.view(np.int64)).cuda() if a.size else torch.zeros(1, dtype=torch.int64, device="cuda")
        dev.append(bq.DeviceRleBitmap(t, 0, a.size))
    ts = sorted({1, n, int(rng.integers(1, n + 1)), max(1, n // 2), max(1, n // 10)})
    accs = [[bool(x) for x in rng.integers(0, 2, size=n + 1)], [k % 2 == 1 for k in range(n + 1)]]
    fails = []
    exp_t = {t: O.cdom_threshold(streams, r, t) for t in ts}
    exp_a = [O.cdom_symmetric(streams, r, a) for a in accs]
    for sliced in ("0", "1"):
        os.environ["BQ_RLE_SLICED"] = sliced
        ranges = [None]
        if tiles > 2:
            b = 1024 * int(rng.integers(0, tiles - 1))
            e = min(nw, b + 1024 * int(rng.integers(1, tiles)))
            ranges.append((b, e))
        for wr in ranges:
            q = bq.RleQuery(dev, r, word_range=wr)
            lo, hi = wr if wr else (0, nw)
            for t in ts:
                out, pc = q.threshold(t)
                got = out[: hi - lo].cpu().numpy().view(np.uint64)
                if not np.array_equal(got, exp_t[t][lo:hi]):
                    fails.append(f"seed {seed} sliced {sliced} range {wr} T {t} n {n} r {r} noncanon {noncanon}")
            for a, e in zip(accs, exp_a):
                out, pc = q.symmetric(a)
                got = out[: hi - lo].cpu().numpy().view(np.uint64)
                if not np.array_equal(got, e[lo:hi]):
                    fails.append(f"seed {seed} sliced {sliced} range {wr} accept n {n} r {r} noncanon {noncanon}")
            q.close()
    return fails


def validate_case(seed):
    """K3's validation against the oracle's decompress on corrupted streams: both must
    accept or both reject (FormatError); accepted streams must decode identically."""
    rng = np.random.default_rng(seed)
    nw = int(rng.choice([1, 3, 40, 1024, 1500, 5000, 40000]))
    r = 64 * nw - (int(rng.integers(0, 64)) if rng.random() < 0.6 else 0)
    r = max(r, 1)
    nw = (r + 63) // 64
    if rng.random() < 0.3 and r % 64 == 0:
        s = noncanonical(rng, nw)
    else:
        s = canonical(rng, r, nw, ["markov", "literal", "sparse", "windows", "short"][int(rng.integers(5))])
    s = s.copy()
    kind = int(rng.integers(7))
    if s.size and kind == 1:
        s = s[: int(rng.integers(0, s.size))]
    elif s.size and kind == 2:  # bump a word's dirty field (a marker's, if it is one)
        i = int(rng.integers(s.size))
        s[i] = np.uint64((int(s[i]) + (int(rng.integers(1, 4)) << 33)) & ((1 << 64) - 1))
    elif s.size and kind == 3:  # bump a run
        i = int(rng.integers(s.size))
        s[i] = np.uint64((int(s[i]) + (int(rng.integers(1, 3000)) << 1)) & ((1 << 64) - 1))
    elif s.size and kind == 4:  # high bits of the last word
        s[-1] = np.uint64(int(s[-1]) | (1 << 63) | (1 << int(rng.integers(64))))
    elif kind == 5:  # one more marker at the end
        s = np.append(s, np.uint64(marker(int(rng.integers(2)), int(rng.integers(0, 3)), 0)))
    elif s.size and kind == 6:  # a random word
        s[int(rng.integers(s.size))] = rng.integers(0, 2**64 - 1, dtype=np.uint64)
    try:
        exp = O.rle_decompress(s, r)
        ok = True
    except O.OracleError:
        ok = False
    t = torch.from_numpy(s.view(np.int64)).cuda() if s.size else torch.zeros(1, dtype=torch.int64, device="cuda")
    d = [bq.DeviceRleBitmap(t, 0, s.size)]
    try:
        q = bq.RleQuery(d, r)
        got_ok = True
    except bq.FormatError:
        got_ok = False
    if ok != got_ok:
        return [f"validate seed {seed} kind {kind} r {r} words {s.size}: oracle {'ok' if ok else 'rejects'}, K3 {'ok' if got_ok else 'rejects'}"]
    if ok:
        os.environ["BQ_RLE_SLICED"] = "0"
        out, _ = q.threshold(1)
        if not np.array_equal(out[:nw].cpu().numpy().view(np.uint64), exp):
            return [f"validate seed {seed} kind {kind} r {r}: decode differs"]
        q.close()
    return []


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    mode = sys.argv[3] if len(sys.argv) > 3 else "eval"
    t0 = time.time()
    cases = bad = 0
    while time.time() - t0 < budget:
        f = validate_case(seed) if mode == "validate" else run_case(seed)
        for line in f:
            print("MISMATCH", line, flush=True)
        bad += bool(f)
        cases += 1
        seed += 1
    print(f"fuzz_rle ({mode}): {cases} cases, {bad} with mismatches, seeds up to {seed - 1}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
