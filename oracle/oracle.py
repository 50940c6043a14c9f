"""CPU oracle for the threshold / symmetric hot path -- TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithms (Kaser & Lemire's ``bitquorum``
package, /root/reference/pkg/src/bitquorum) so tests can check the CUDA path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import it.  The product
package never does.

Two layers:

* pure-Python restatements of ``oracle.py`` (``brute_threshold``,
  ``brute_symmetric``; reference ``oracle.py:56-80``) for small cases, and
* numpy wrappers over ``liboracle.so`` (``bq_oracle.c``) for word arrays:
  ScanCount, the CSV/wide-OR/wide-AND CPU port, RLE compress/decompress and
  the cdom run sweep.

Parity pin: ``tests/golden/`` holds inputs and outputs produced by running the
reference itself (``tests/golden/make_golden.py``); ``tests/test_oracle.py``
checks every function here against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from collections import Counter
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_LIB_AVX512 = os.path.join(_HERE, "_build", "liboracle_avx512.so")


def _has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fp:
            for line in fp:
                if line.startswith("flags"):
                    return " avx512f " in line + " "
    except OSError:
        pass
    return False
_lib = None

OK, EINPUT, ERESOURCE, EFORMAT = 0, -1, -2, -3


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile bq_oracle.c with the Makefile next to it (gcc, OpenMP)."""
    src = os.path.join(_HERE, "bq_oracle.c")
    if force or any(not os.path.exists(f) or os.path.getmtime(f) < os.path.getmtime(src) for f in (_LIB_PATH, _LIB_AVX512)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        path = _LIB_AVX512 if (_has_avx512() and os.path.exists(_LIB_AVX512)
                               and os.environ.get("BQ_ORACLE_AVX512", "1") != "0") else _LIB_PATH
        L = ctypes.CDLL(path)
        L._bq_path = path
        P = ctypes.c_void_p
        U64 = ctypes.c_uint64
        I = ctypes.c_int
        L.orc_scan_count.argtypes = [P, P, I, U64, I, P]
        L.orc_scan_count_symmetric.argtypes = [P, P, I, U64, P, P]
        L.orc_threshold_port.argtypes = [P, P, I, U64, I, P, I]
        L.orc_symmetric_port.argtypes = [P, P, I, U64, P, P, I]
        L.orc_rle_decompress.argtypes = [P, U64, U64, P]
        L.orc_rle_compress.argtypes = [P, U64, U64, P, U64, P]
        L.orc_cdom_threshold.argtypes = [P, P, I, U64, I, P, P]
        L.orc_cdom_symmetric.argtypes = [P, P, I, U64, P, P, P]
        L.orc_num_threads.argtypes = []
        L.orc_gen_bernoulli.argtypes = [U64, ctypes.c_uint32, ctypes.c_uint32, U64, U64, P]
        L.orc_gen_density_q16.argtypes = [U64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_gen_density_q16.restype = ctypes.c_uint32
        L.orc_gen_markov_rle.argtypes = [U64, ctypes.c_uint32, U64, ctypes.c_double, ctypes.c_double, P, U64, P]
        for name in ("orc_scan_count", "orc_scan_count_symmetric", "orc_threshold_port",
                     "orc_symmetric_port", "orc_rle_decompress", "orc_rle_compress",
                     "orc_cdom_threshold", "orc_cdom_symmetric", "orc_num_threads", "orc_gen_bernoulli",
                     "orc_gen_markov_rle"):
            getattr(L, name).restype = I
        _lib = L
    return _lib


def word_count(bits: int) -> int:
    return (bits + 63) // 64


# ---------------------------------------------------------------------------
# pure-Python restatement of reference oracle.py:56-80

def brute_threshold(position_sets: Sequence[Iterable[int]], t: int) -> list[int]:
    """Positions occurring in at least ``t`` sets (reference oracle.py:56-65)."""
    n = len(position_sets)
    if not 1 <= t <= n:
        raise ValueError(f"threshold {t} outside [1, {n}]")
    counts: Counter = Counter()
    for s in position_sets:
        for p in s:
            counts[p] += 1
    return sorted(p for p, c in counts.items() if c >= t)


def brute_symmetric(position_sets: Sequence[Iterable[int]], accept: Sequence[bool],
                    universe: int) -> list[int]:
    """Positions p < universe with accept[count(p)] (reference oracle.py:68-80)."""
    if len(accept) - 1 != len(position_sets):
        raise ValueError("accept length must be N + 1")
    counts: Counter = Counter()
    for s in position_sets:
        for p in s:
            counts[p] += 1
    if accept[0]:
        return [p for p in range(universe) if accept[counts.get(p, 0)]]
    return sorted(p for p, c in counts.items() if accept[c])


def positions_of(words: np.ndarray) -> list[int]:
    words = np.asarray(words, dtype=np.uint64)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    return np.flatnonzero(bits).tolist()


def words_from_positions(positions: Iterable[int], r: int) -> np.ndarray:
    out = np.zeros(word_count(r), dtype=np.uint64)
    for p in positions:
        out[p >> 6] |= np.uint64(1 << (p & 63))
    return out


# ---------------------------------------------------------------------------
# numpy wrappers over liboracle.so

def _as_inputs(inputs: Sequence[np.ndarray]):
    arrs = [np.ascontiguousarray(a, dtype=np.uint64) for a in inputs]
    n = len(arrs)
    ptrs = (ctypes.c_void_p * max(n, 1))(*[a.ctypes.data if a.size else 0 for a in arrs])
    lens = (ctypes.c_uint64 * max(n, 1))(*[a.size for a in arrs])
    return arrs, ptrs, lens, n


def _check(rc: int, what: str):
    if rc != OK:
        raise OracleError(rc, what)


def scan_count(inputs: Sequence[np.ndarray], r: int, t: int) -> np.ndarray:
    """ScanCount (reference counters.py:46-67) -> word_count(r) words."""
    arrs, ptrs, lens, n = _as_inputs(inputs)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    _check(lib().orc_scan_count(ptrs, lens, n, r, t, out.ctypes.data), "scan_count")
    return out[: word_count(r)]


def scan_count_symmetric(inputs: Sequence[np.ndarray], r: int, accept: Sequence[bool]) -> np.ndarray:
    """scan_count_symmetric (reference counters.py:70-83)."""
    arrs, ptrs, lens, n = _as_inputs(inputs)
    acc = np.asarray([1 if a else 0 for a in accept], dtype=np.uint8)
    if acc.size != n + 1:
        raise ValueError("accept length must be N + 1")
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    _check(lib().orc_scan_count_symmetric(ptrs, lens, n, r, acc.ctypes.data, out.ctypes.data),
           "scan_count_symmetric")
    return out[: word_count(r)]


def threshold_port(inputs: Sequence[np.ndarray], r: int, t: int, threads: int = 0) -> np.ndarray:
    """Multi-threaded CPU port: wide_or / wide_and / csv_threshold (bitparallel.py:51-129)."""
    arrs, ptrs, lens, n = _as_inputs(inputs)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    _check(lib().orc_threshold_port(ptrs, lens, n, r, t, out.ctypes.data, threads), "threshold_port")
    return out[: word_count(r)]


def symmetric_port(inputs: Sequence[np.ndarray], r: int, accept: Sequence[bool],
                   threads: int = 0) -> np.ndarray:
    arrs, ptrs, lens, n = _as_inputs(inputs)
    acc = np.asarray([1 if a else 0 for a in accept], dtype=np.uint8)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    _check(lib().orc_symmetric_port(ptrs, lens, n, r, acc.ctypes.data, out.ctypes.data, threads),
           "symmetric_port")
    return out[: word_count(r)]


def rle_decompress(stream: np.ndarray, r: int) -> np.ndarray:
    """decompress (reference bitmaps.py:417-431); raises OracleError(EFORMAT)."""
    s = np.ascontiguousarray(stream, dtype=np.uint64)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    _check(lib().orc_rle_decompress(s.ctypes.data if s.size else 0, s.size, r, out.ctypes.data),
           "rle_decompress")
    return out[: word_count(r)]


def rle_compress(words: np.ndarray, r: int) -> np.ndarray:
    """compress (reference bitmaps.py:407-414), canonical RleBuilder encoding."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    cap = 2 * w.size + 8
    out = np.zeros(cap, dtype=np.uint64)
    n_out = ctypes.c_uint64(0)
    _check(lib().orc_rle_compress(w.ctypes.data if w.size else 0, w.size, r, out.ctypes.data, cap,
                                  ctypes.byref(n_out)), "rle_compress")
    return out[: n_out.value].copy()


_BRANCHES = ("or", "and", "looped", "scan")


def cdom_threshold(streams: Sequence[np.ndarray], r: int, t: int, stats: dict | None = None) -> np.ndarray:
    """cdom_threshold (reference runmerge.py:198-241), output uncompressed.  ``stats``
    is filled as the reference fills it: untouched for T = 1 / T = N (wide_or /
    wide_and, :203-206) and r = 0 (:209-210), else segments, heap_pops and the
    dirty-segment dispatch counts under ``branches`` (nonzero keys only, :237-240)."""
    arrs, ptrs, lens, n = _as_inputs(streams)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    st = np.zeros(6, dtype=np.uint64)
    _check(lib().orc_cdom_threshold(ptrs, lens, n, r, t, out.ctypes.data, st.ctypes.data),
           "cdom_threshold")
    if stats is not None and 1 < t < n and word_count(r):
        stats["segments"] = int(st[0])
        stats["heap_pops"] = int(st[1])
        stats["branches"] = {b: int(c) for b, c in zip(_BRANCHES, st[2:]) if c}
    return out[: word_count(r)]


def cdom_symmetric(streams: Sequence[np.ndarray], r: int, accept: Sequence[bool],
                   stats: dict | None = None) -> np.ndarray:
    """cdom_symmetric (reference runmerge.py:244-299), output uncompressed; ``stats``
    gets segments and heap_pops (:296-298) unless r = 0."""
    arrs, ptrs, lens, n = _as_inputs(streams)
    acc = np.asarray([1 if a else 0 for a in accept], dtype=np.uint8)
    out = np.zeros(max(word_count(r), 1), dtype=np.uint64)
    st = np.zeros(6, dtype=np.uint64)
    _check(lib().orc_cdom_symmetric(ptrs, lens, n, r, acc.ctypes.data, out.ctypes.data,
                                    st.ctypes.data), "cdom_symmetric")
    if stats is not None and word_count(r):
        stats["segments"] = int(st[0])
        stats["heap_pops"] = int(st[1])
    return out[: word_count(r)]


def num_threads() -> int:
    return lib().orc_num_threads()


def trim(words: np.ndarray) -> np.ndarray:
    """Drop trailing zero words, as UncompressedBitmap.__init__ does (bitmaps.py:66-67)."""
    w = np.asarray(words, dtype=np.uint64)
    nz = np.flatnonzero(w)
    return w[: (nz[-1] + 1) if nz.size else 0]


# ---------------------------------------------------------------------------
# benchmark input generators (independent restatement of csrc/bq_gen.h; used by
# bench.py's CPU legs so they never load libbq.so)

def gen_bernoulli(seed: int, bitmap: int, q16: int, w0: int, nw: int) -> np.ndarray:
    """Words [w0, w0 + nw) of bitmap ``bitmap``, each bit Bernoulli(q16 / 2^16)."""
    out = np.empty(max(nw, 1), dtype=np.uint64)
    _check(lib().orc_gen_bernoulli(seed, bitmap, q16, w0, nw, out.ctypes.data), "gen_bernoulli")
    return out[:nw]


def gen_density_q16(seed: int, bitmap: int, lo: int, hi: int) -> int:
    return int(lib().orc_gen_density_q16(seed, bitmap, lo, hi))


def gen_markov_rle(seed: int, bitmap: int, r: int, mean_one: float, mean_zero: float) -> np.ndarray:
    """C4 stream: geometric one / zero runs of the given means, canonical RLE."""
    cap = max(4096, r // 64 // 4)
    while True:
        out = np.empty(cap, dtype=np.uint64)
        n = ctypes.c_uint64(0)
        rc = lib().orc_gen_markov_rle(seed, bitmap, r, float(mean_one), float(mean_zero), out.ctypes.data, cap,
                                      ctypes.byref(n))
        if rc == ERESOURCE:
            cap = int(n.value) + 16
            continue
        _check(rc, "gen_markov_rle")
        return out[: n.value].copy()


def library_path() -> str:
    """The oracle library in use (AVX-512 build on hosts with avx512f)."""
    return lib()._bq_path
