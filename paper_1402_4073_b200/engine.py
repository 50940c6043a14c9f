"""Device-side engine: prepared queries over HBM-resident inputs, the upload
cache for immutable host bitmaps, and the host-buffer streaming sweep.

Everything here calls libbq.so through ctypes (``_lib``); torch is used only
for device memory and streams.
"""

from __future__ import annotations

import ctypes
import os
from array import array
from itertools import chain
import threading
from collections import OrderedDict
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .bitmaps import DeviceBitmap, DeviceRleBitmap, word_count
from .errors import InputError


def _device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise _lib.ExtensionMissing("no CUDA device is visible; the bitmap engine has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise InputError(f"device must be a CUDA device, got {d}")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def stream_handle(stream=None, device=None) -> int:
    s = torch.cuda.current_stream(device) if stream is None else stream
    return int(s.cuda_stream)


def host_words(b) -> np.ndarray:
    """A host bitmap's words as a uint64 numpy array (no copy when already numpy)."""
    w = b.words
    if isinstance(w, np.ndarray):
        return np.ascontiguousarray(w, dtype=np.uint64)
    # the reference keeps words as a list of Python ints (bitmaps.py:54-72); array('Q')
    # packs them ~1.7x faster than numpy's per-object conversion, same range check
    try:
        return np.frombuffer(array("Q", w), dtype=np.uint64)
    except (TypeError, OverflowError):
        return np.array(w, dtype=np.uint64)


def to_device_words(arr: np.ndarray, device) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint64).view(np.int64))
    return t.to(device, non_blocking=False)


class UploadCache:
    """Device copies of immutable host bitmaps, keyed by object identity.

    The reference's bitmaps are immutable (bitmaps.py:12-13) and its harness
    passes the same object several times for replicated inputs
    (bench/similarity.py:53-55), deduplicating by id() (competitions.py:259-262);
    this cache does the same.  Entries hold a strong reference to the host object
    so its id cannot be reused while cached.  LRU-bounded by device bytes
    (env BQ_UPLOAD_CACHE_BYTES, default 8 GiB).
    """

    def __init__(self, max_bytes: int | None = None):
        self.max_bytes = int(os.environ.get("BQ_UPLOAD_CACHE_BYTES", 8 << 30)) if max_bytes is None else max_bytes
        self._d: OrderedDict = OrderedDict()
        self._bytes = 0
        self._lock = threading.Lock()

    def get(self, b, device: torch.device) -> torch.Tensor:
        key = (id(b), device.index)
        with self._lock:
            hit = self._d.get(key)
            if hit is not None and hit[0] is b:
                self._d.move_to_end(key)
                return hit[1]
        t = to_device_words(host_words(b), device)
        nbytes = t.numel() * 8
        with self._lock:
            if nbytes <= self.max_bytes:
                self._d[key] = (b, t)
                self._bytes += nbytes
                while self._bytes > self.max_bytes and self._d:
                    _, (_, old) = self._d.popitem(last=False)
                    self._bytes -= old.numel() * 8
        return t

    def clear(self):
        with self._lock:
            self._d.clear()
            self._bytes = 0


UPLOADS = UploadCache()


def _check_out(out, out_words: int, device) -> None:
    """A caller-supplied result buffer: on the query's device, 64-bit words,
    contiguous, at least ``out_words`` long and 16-byte aligned (the kernels store
    128-bit vectors; include/bq.h)."""
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.device != device:
        raise InputError(f"output tensor must be a CUDA tensor on {device}")
    if out.dtype not in (torch.int64, torch.uint64) or not out.is_contiguous():
        raise InputError("output tensor must be a contiguous int64/uint64 tensor")
    if out.numel() < out_words:
        raise InputError(f"output tensor holds {out.numel()} words, the result needs {out_words}")
    if out.data_ptr() % 16:
        raise InputError("output tensor must be 16-byte aligned")


class ThresholdQuery:
    """A prepared query (``bq_query``) over N device-resident uncompressed inputs.

    ``inputs``: DeviceBitmap objects or 1-D int64 CUDA tensors (all words valid).
    ``word_range``: evaluate only output words [begin, end) (a shard); ``begin``
    must be even.  The pointer table is uploaded once; each ``threshold`` /
    ``symmetric`` call is a single kernel launch on ``stream``.
    """

    def __init__(self, inputs: Sequence, r_bits: int, word_range=None, device=None):
        self._lib = _lib.load()
        self.device = _device(device if device is not None else self._infer_device(inputs))
        self.n = len(inputs)
        self.r_bits = int(r_bits)
        self._keep = []
        pairs = []
        for x in inputs:
            if isinstance(x, DeviceBitmap):
                t, n_words = x.data, x.n_words
            elif isinstance(x, torch.Tensor):
                t, n_words = x, x.numel()
            else:
                raise InputError(f"ThresholdQuery needs device inputs, got {type(x).__name__}")
            if not t.is_cuda or t.dtype not in (torch.int64, torch.uint64):
                raise InputError("device inputs must be int64/uint64 CUDA tensors")
            if n_words and not t.is_contiguous():
                raise InputError("device inputs must be contiguous")
            self._keep.append(t)
            pairs.append((t.data_ptr() if n_words else 0, n_words))
        begin, end = (0, (1 << 64) - 1) if word_range is None else (int(word_range[0]), int(word_range[1]))
        self._spans = _lib.spans(pairs)
        h = ctypes.c_void_p()
        _lib.check(self._lib.bq_query_create(self._spans.ctypes.data, self.n, self.r_bits, begin, end,
                                             self.device.index, ctypes.byref(h)), "bq_query_create")
        self._h = h
        self.out_words = int(self._lib.bq_query_out_words(h))

    @staticmethod
    def _infer_device(inputs):
        for x in inputs:
            d = x.data.device if isinstance(x, DeviceBitmap) else getattr(x, "device", None)
            if d is not None and d.type == "cuda":
                return d
        return None

    def _outs(self, out, popcnt, last_nz):
        if out is None:
            out = torch.empty(max(self.out_words, 1), dtype=torch.int64, device=self.device)
        else:
            _check_out(out, self.out_words, self.device)
        if popcnt is None:
            popcnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        return out, popcnt, last_nz

    def threshold(self, t: int, out=None, popcnt=None, last_nz=None, stream=None):
        """Launch theta(t): returns (out, popcnt); popcnt is ADDED to (zeroed if allocated here)."""
        out, popcnt, last_nz = self._outs(out, popcnt, last_nz)
        _lib.check(self._lib.bq_query_threshold(
            self._h, int(t), out.data_ptr(), popcnt.data_ptr(),
            last_nz.data_ptr() if last_nz is not None else None,
            stream_handle(stream, self.device)), "bq_query_threshold")
        return out, popcnt

    def symmetric(self, accept, out=None, popcnt=None, last_nz=None, stream=None):
        acc = accept_bytes(accept, self.n)
        out, popcnt, last_nz = self._outs(out, popcnt, last_nz)
        _lib.check(self._lib.bq_query_symmetric(
            self._h, acc.ctypes.data, out.data_ptr(), popcnt.data_ptr(),
            last_nz.data_ptr() if last_nz is not None else None,
            stream_handle(stream, self.device)), "bq_query_symmetric")
        return out, popcnt

    def close(self):
        if getattr(self, "_h", None):
            self._lib.bq_query_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RleQuery:
    """A prepared query over N device-resident RLE streams (``bq_rle_query``).

    Creation decodes every stream's marker chain on the device into a tile
    directory (K3) and validates the encoding (FormatError).  ``word_range``
    (begin, end) restricts the output to result words [begin, end) -- one rank's
    shard (``shard.ShardedQuery``); the streams stay whole (replicated)."""

    def __init__(self, streams: Sequence, r_bits: int, device=None, word_range=None):
        self._lib = _lib.load()
        first = streams[0] if streams else None
        d = first.data.device if isinstance(first, DeviceRleBitmap) else getattr(first, "device", None)
        self.device = _device(device if device is not None else d)
        self.n = len(streams)
        self.r_bits = int(r_bits)
        # one pass per column (a fresh query over 1024 streams is ~1 ms of device work,
        # so the marshalling stays vectorised: no per-stream ctypes structs)
        try:  # all DeviceRleBitmap: their cached (pointer, words) pairs, one pass
            pairs = [s.span() for s in streams]
            self._keep = [s.data for s in streams]
        except AttributeError:
            ts = [s.data if isinstance(s, DeviceRleBitmap) else s for s in streams]
            nws = [s.n_words if isinstance(s, DeviceRleBitmap) else s.numel() for s in streams]
            if not all(isinstance(t, torch.Tensor) and t.is_cuda for t in ts):
                raise InputError("RLE streams must be CUDA tensors")
            self._keep = ts
            pairs = [(t.data_ptr() if n else 0, n) for t, n in zip(ts, nws)]
        self._spans = (np.fromiter(chain.from_iterable(pairs), dtype=np.uint64, count=2 * len(pairs)).reshape(-1, 2)
                       if pairs else np.zeros((1, 2), dtype=np.uint64))
        self._create(word_range)

    @classmethod
    def from_packed(cls, flat, offsets, lengths, r_bits: int, device=None, word_range=None):
        """A query over streams packed in one device tensor: stream i is
        ``flat[offsets[i] : offsets[i] + lengths[i]]`` (words).  No per-stream Python
        objects: the span table is computed with numpy (a BQDS-style dataset or a
        batch of uploaded streams)."""
        if not isinstance(flat, torch.Tensor) or not flat.is_cuda or flat.dtype not in (torch.int64, torch.uint64):
            raise InputError("packed streams must be an int64/uint64 CUDA tensor")
        offs = np.asarray(offsets, dtype=np.uint64)
        lens = np.asarray(lengths, dtype=np.uint64)
        if offs.shape != lens.shape or offs.ndim != 1:
            raise InputError("offsets and lengths must be 1-D and of equal length")
        if offs.size and int((offs + lens).max()) > flat.numel():
            raise InputError("a packed stream extends past the buffer")
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self.device = _device(device if device is not None else flat.device)
        self.n = int(offs.size)
        self.r_bits = int(r_bits)
        self._keep = [flat]
        ptrs = np.where(lens > 0, np.uint64(flat.data_ptr()) + offs * np.uint64(8), np.uint64(0))
        self._spans = _lib.span_columns(ptrs, lens)
        self._create(word_range)
        return self

    def _create(self, word_range):
        h = ctypes.c_void_p()
        w0, w1 = word_range if word_range is not None else (0, word_count(self.r_bits))
        _lib.check(self._lib.bq_rle_query_create_range(self._spans.ctypes.data, self.n, self.r_bits, int(w0), int(w1),
                                                       self.device.index, ctypes.byref(h)), "bq_rle_query_create")
        self._h = h
        self.word_range = (int(w0), int(w0) + int(self._lib.bq_rle_query_out_words(h)))
        self.out_words = self.word_range[1] - self.word_range[0]

    @property
    def directory_bytes(self) -> int:
        return int(self._lib.bq_rle_query_directory_bytes(self._h))

    @property
    def layout_stats(self) -> tuple:
        """(markers, literal words) of the tile-sliced layout; (0, 0) until it is built."""
        m, l = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _lib.check(self._lib.bq_rle_query_layout_stats(self._h, ctypes.byref(m), ctypes.byref(l)),
                   "bq_rle_query_layout_stats")
        return int(m.value), int(l.value)

    @property
    def layout_events(self) -> int:
        """Difference-array events of the tile-sliced layout (16-bit each, phase A's input); 0 until built."""
        e = ctypes.c_uint64(0)
        _lib.check(self._lib.bq_rle_query_layout_events(self._h, ctypes.byref(e)), "bq_rle_query_layout_events")
        return int(e.value)

    def sweep_stats(self, t: int = 0, stream=None) -> dict:
        """The counters cdom's CPU sweep reports (runmerge.py:237-240, :296-298),
        recomputed on the device from the inputs' merged runs (K8): segments,
        heap_pops and, for a threshold t > 0, the dirty-segment dispatch counts
        (nonzero keys only, like the reference's ``branches`` dict)."""
        st = np.zeros(6, dtype=np.uint64)
        _lib.check(self._lib.bq_rle_query_sweep_stats(self._h, int(t), st.ctypes.data,
                                                      stream_handle(stream, self.device)),
                   "bq_rle_query_sweep_stats")
        res = {"segments": int(st[0]), "heap_pops": int(st[1])}
        if t > 0:
            res["branches"] = {b: int(c) for b, c in zip(("or", "and", "looped", "scan"), st[2:]) if c}
        return res

    def _outs(self, out, popcnt):
        if out is None:
            out = torch.empty(max(self.out_words, 1), dtype=torch.int64, device=self.device)
        else:
            _check_out(out, self.out_words, self.device)
        if popcnt is None:
            popcnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        return out, popcnt

    def threshold(self, t: int, out=None, popcnt=None, stream=None):
        out, popcnt = self._outs(out, popcnt)
        _lib.check(self._lib.bq_rle_query_threshold(self._h, int(t), out.data_ptr(), popcnt.data_ptr(),
                                                    stream_handle(stream, self.device)),
                   "bq_rle_query_threshold")
        return out, popcnt

    def symmetric(self, accept, out=None, popcnt=None, stream=None):
        acc = accept_bytes(accept, self.n)
        out, popcnt = self._outs(out, popcnt)
        _lib.check(self._lib.bq_rle_query_symmetric(self._h, acc.ctypes.data, out.data_ptr(),
                                                    popcnt.data_ptr(), stream_handle(stream, self.device)),
                   "bq_rle_query_symmetric")
        return out, popcnt

    def close(self):
        if getattr(self, "_h", None):
            self._lib.bq_rle_query_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def release_cached_memory() -> None:
    """Return the device memory libbq keeps for later queries (RLE directories,
    tile-sliced layouts and their build scratch come from a pool that retains up
    to 16 GiB after frees) to the driver (bq_release_cached_memory)."""
    _lib.check(_lib.load().bq_release_cached_memory(), "bq_release_cached_memory")


def accept_bytes(accept, n: int) -> np.ndarray:
    """SymmetricSpec (``.accept``) or a bool sequence -> n + 1 bytes (oracle.py:17-31)."""
    acc = getattr(accept, "accept", accept)
    arr = np.asarray([1 if a else 0 for a in acc], dtype=np.uint8)
    if arr.size != n + 1:
        raise InputError(f"spec arity {arr.size - 1} != {n} inputs")  # counters.py:73-74
    return arr


def sweep_host(inputs: Sequence[np.ndarray], r_bits: int, queries: Sequence, outs=None,
               device=None, chunk_words: int = 0):
    """End-to-end path over HOST word arrays (ideally pinned).

    ``queries``: ints (thresholds) or accept vectors.  Results land in ``outs``
    (list of uint64 numpy arrays of word_count(r_bits) words; allocated if None).
    Inputs are streamed through the GPU in word-range chunks with copy-in,
    compute and copy-out overlapped (bq_sweep_host).  Returns (outs, popcounts).
    """
    lib = _lib.load()
    dev = _device(device)
    n, nq = len(inputs), len(queries)
    nw = word_count(int(r_bits))
    arrs = [np.asarray(a) for a in inputs]
    for a in arrs:
        if a.dtype not in (np.uint64, np.int64) or not a.flags.c_contiguous:
            raise InputError("host inputs must be contiguous uint64 arrays")
    ptrs = (ctypes.c_void_p * n)(*[a.ctypes.data if a.size else None for a in arrs])
    lens = (ctypes.c_uint64 * n)(*[a.size for a in arrs])
    ts = (ctypes.c_int * nq)()
    acc = np.zeros((nq, n + 1), dtype=np.uint8)
    for k, q in enumerate(queries):
        if isinstance(q, (int, np.integer)):
            ts[k] = int(q)
            if not 1 <= int(q) <= n:
                raise InputError(f"threshold {int(q)} outside [1, {n}]")
        else:
            ts[k] = 0
            acc[k] = accept_bytes(q, n)
    if outs is None:
        outs = [np.empty(nw, dtype=np.uint64) for _ in range(nq)]
    optrs = (ctypes.c_void_p * nq)(*[o.ctypes.data for o in outs])
    pops = (ctypes.c_ulonglong * nq)()
    _lib.check(lib.bq_sweep_host(ptrs, lens, n, int(r_bits), ts, acc.ctypes.data, nq, optrs, pops,
                                 dev.index, int(chunk_words)), "bq_sweep_host")
    return outs, [int(p) for p in pops]
