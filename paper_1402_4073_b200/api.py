"""Drop-in entry points with the reference's names and signatures.

Each function mirrors one reference callable on the threshold / symmetric path
(paths relative to /root/reference/pkg/src/bitquorum/) and evaluates it on the
B200 through libbq.so.  Inputs may be the reference's own bitmap objects, this
package's mirrors (``bitmaps.UncompressedBitmap`` / ``RleBitmap``), or
HBM-resident ``DeviceBitmap`` / ``DeviceRleBitmap``:

* host inputs are uploaded once (identity-keyed cache) and the result comes
  back as ``type(bitmaps[0])`` with the reference's trimming; RLE inputs give
  a canonically encoded RLE result (counters.py:33-37, runmerge.py:241);
* device inputs give a device result (no host round trip).

All the reference's algorithm variants compute the same function, so they all
dispatch to the same kernels; they differ only in their argument contracts and
``stats`` keys.  Keys that describe the query (counter_width, increments,
bitmap_ops) are reproduced; cdom's keys count the steps of its CPU heap sweep
(segments, heap_pops, branches; runmerge.py:238-240): the device path does not
take that sweep, so they are recomputed from the inputs' merged runs by a
separate device pass (K8), only when a ``stats`` dict is passed.  There is no CPU fallback:
without the CUDA library every call raises ``ExtensionMissing``.
"""

from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .bitmaps import DeviceBitmap, DeviceRleBitmap, RleBitmap, UncompressedBitmap, kind_of, word_count
from .engine import UPLOADS, RleQuery, ThresholdQuery, accept_bytes, host_words, to_device_words
from .errors import InputError, ResourceError

DEFAULT_BUDGET_BYTES = 1 << 30  # counters.py:18


def counter_width(n: int) -> int:
    """Counter width the reference's ScanCount would use (counters.py:21-27)."""
    if n < 128:
        return 8
    if n < 1 << 15:
        return 16
    return 32


def weight_bits(n: int) -> int:
    """m = floor(log2 2N): bits of the device's bit-sliced counter (circuits/core.py:240-242)."""
    return (2 * n).bit_length() - 1


def looped_op_count(n: int, t: int) -> int:
    """Closed form of Looped's binary-op count (circuits/bitparallel.py:46-48)."""
    return 2 * n * t - n - t * t + t - 1


def csv_op_count(n: int, t: int) -> int:
    """Number of counted bitmap ops csv_threshold issues (circuits/bitparallel.py:84-121):
    5 per digit update on the trailing-zeros schedule, 5 per digit of the
    redundant-to-binary pass and 1 per digit of the comparator."""
    m = weight_bits(n)
    ops = 0
    time = 1
    for _ in range(2, n):
        time += 1
        ops += 5 * ((time & -time).bit_length() - 1)
    return ops + 6 * m


def _check_t(n: int, t: int):
    if not 1 <= t <= n:
        raise InputError(f"threshold {t} outside [1, {n}]")  # counters.py:40-43


def _classify(bitmaps) -> str:
    if not bitmaps:
        raise InputError("need at least one input bitmap")
    kinds = {kind_of(b) for b in bitmaps}
    if kinds <= {"u", "du"}:
        return "u"
    if kinds <= {"r", "dr"}:
        return "r"
    raise InputError("mixed bitmap representations; convert explicitly with compress/decompress")


def _device_for(bitmaps):
    for b in bitmaps:
        if isinstance(b, (DeviceBitmap, DeviceRleBitmap)):
            return b.data.device
    return torch.device("cuda", torch.cuda.current_device())


def _dev_inputs(bitmaps, device):
    out = []
    for b in bitmaps:
        k = kind_of(b)
        if k in ("du", "dr"):
            out.append(b)
        else:
            t = UPLOADS.get(b, device)
            out.append(DeviceBitmap(t, b.bit_length, t.numel()) if k == "u" else
                       DeviceRleBitmap(t, b.bit_length, t.numel()))
    return out


class _QueryCache:
    """Prepared queries (device pointer table; for RLE inputs also the K3 tile
    directory) keyed by the identities of their input objects.  Bitmaps are
    immutable after construction (reference bitmaps.py:12-13), so a query stays
    valid as long as its inputs live; entries hold strong references to them so
    ids cannot be reused.  LRU-bounded by entry count and by the device bytes of
    the uploaded host inputs the cached queries keep alive (the upload cache's
    bound, BQ_UPLOAD_CACHE_BYTES): a query holds its inputs' device copies, so
    without the second bound evicted uploads would outlive the upload cache."""

    def __init__(self, maxsize: int = 32, max_bytes: int | None = None):
        from collections import OrderedDict
        import threading

        self.maxsize = maxsize
        self._max_bytes = max_bytes
        self._d = OrderedDict()
        self._bytes = 0
        self._lock = threading.Lock()

    @property
    def max_bytes(self) -> int:
        return UPLOADS.max_bytes if self._max_bytes is None else self._max_bytes

    @property
    def held_bytes(self) -> int:
        return self._bytes

    def get(self, kind: str, bitmaps, r: int, device):
        key = (kind, tuple(id(b) for b in bitmaps), r, device.index)
        with self._lock:
            hit = self._d.get(key)
            if hit is not None and all(x is y for x, y in zip(hit[0], bitmaps)):
                self._d.move_to_end(key)
                return hit[1]
        dev = _dev_inputs(bitmaps, device)
        q = ThresholdQuery(dev, r, device=device) if kind == "u" else RleQuery(dev, r, device=device)
        # device bytes of uploaded host inputs (device-resident inputs belong to the caller)
        seen, nbytes = set(), 0
        for b, d in zip(bitmaps, dev):
            if kind_of(b) in ("u", "r") and id(d.data) not in seen:
                seen.add(id(d.data))
                nbytes += d.data.numel() * 8
        with self._lock:
            old = self._d.pop(key, None)
            if old is not None:
                self._bytes -= old[2]
            self._d[key] = (list(bitmaps), q, nbytes)
            self._bytes += nbytes
            while self._d and (len(self._d) > self.maxsize or (self._bytes > self.max_bytes and len(self._d) > 1)):
                _, (_, _, nb) = self._d.popitem(last=False)
                self._bytes -= nb
        return q

    def clear(self):
        with self._lock:
            self._d.clear()
            self._bytes = 0


QUERIES = _QueryCache()


def compress_words(words, bit_length: int) -> list:
    """Canonical RLE encoding of uncompressed words (RleBuilder, bitmaps.py:351-414)."""
    lib = _lib.load()
    arr = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    nw = word_count(bit_length)
    if arr.size > nw:
        raise InputError("more words than bit_length allows")
    cap = 2 * arr.size + 8
    out = np.empty(cap, dtype=np.uint64)
    n_out = ctypes.c_uint64(0)
    _lib.check(lib.bq_rle_encode_host(arr.ctypes.data if arr.size else None, arr.size, bit_length,
                                      out.ctypes.data, cap, ctypes.byref(n_out)), "bq_rle_encode_host")
    return out[: n_out.value].tolist()


def _encode_on_device(words: torch.Tensor, bit_length: int):
    """K7 (bq_rle_encode_device): canonical stream of device words -> (device buffer, length)."""
    lib = _lib.load()
    nw = word_count(bit_length)
    cap = nw + 2
    dout = torch.empty(max(cap, 2), dtype=torch.int64, device=words.device)
    n_out = ctypes.c_uint64(0)
    _lib.check(lib.bq_rle_encode_device(words.data_ptr() if words.numel() else None, min(words.numel(), nw),
                                        bit_length, dout.data_ptr(), cap, ctypes.byref(n_out),
                                        torch.cuda.current_stream(words.device).cuda_stream), "bq_rle_encode_device")
    return dout, int(n_out.value)


def encode_device(words: torch.Tensor, bit_length: int) -> np.ndarray:
    """Canonical RLE encoding (RleBuilder, bitmaps.py:351-414) of device words,
    computed on the GPU (bq_rle_encode_device); returns the host stream."""
    dout, n = _encode_on_device(words, bit_length)
    return dout[:n].cpu().numpy().view(np.uint64)


def compress_device(bitmap, device=None) -> DeviceRleBitmap:
    """bitmaps.compress (bitmaps.py:407-414) with the result kept in HBM: the
    canonical stream of an uncompressed bitmap, encoded on the device (K7)."""
    k = kind_of(bitmap)
    if k == "dr":
        return bitmap
    if k == "r":
        return to_device(bitmap, device)
    b = to_device(bitmap, device)
    dout, n = _encode_on_device(b.data[: b.n_words], b.bit_length)
    return DeviceRleBitmap(dout[: max(n, 1)], b.bit_length, n)


def _finish(bitmaps, out: torch.Tensor, nwords: int, r: int, popcnt: torch.Tensor, last_nz: torch.Tensor):
    """Wrap a device result like the reference would (type of bitmaps[0])."""
    proto = bitmaps[0]
    k = kind_of(proto)
    if k == "du":
        return DeviceBitmap(out[:nwords] if nwords else out[:0], r, nwords)
    if k == "dr":
        return DeviceBitmap(out[:nwords] if nwords else out[:0], r, nwords)
    if k == "u":
        used = int(last_nz.item())
        res = type(proto)(out[:used].cpu().numpy().view(np.uint64).tolist(), r)
    else:  # RLE in -> canonical RLE out, encoded on the device; only the stream crosses PCIe
        res = type(proto)(encode_device(out[:nwords], r).tolist(), r)
    card = int(popcnt.item())
    if hasattr(res, "_card"):
        try:
            res._card = card
        except AttributeError:
            pass
    return res


def _run(bitmaps, r, t=None, accept=None):
    kind = _classify(bitmaps)
    n = len(bitmaps)
    if r is None:
        r = max(b.bit_length for b in bitmaps)
    device = _device_for(bitmaps)
    q = QUERIES.get(kind, bitmaps, r, device)
    nw = word_count(r)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device=device)
    popcnt = torch.zeros(1, dtype=torch.int64, device=device)
    last_nz = torch.zeros(1, dtype=torch.int64, device=device)
    if kind == "u":
        if accept is None:
            q.threshold(t, out, popcnt, last_nz)
        else:
            q.symmetric(accept, out, popcnt, last_nz)
    else:
        if accept is None:
            q.threshold(t, out, popcnt)
        else:
            q.symmetric(accept, out, popcnt)
    return _finish(bitmaps, out, nw, r, popcnt, last_nz)


# ---------------------------------------------------------------------------
# reference entry points


def threshold(bitmaps: Sequence, t: int, r: int | None = None):
    """theta(t; bitmaps) for either representation; result of type(bitmaps[0])."""
    _check_t(len(bitmaps), t)
    return _run(bitmaps, r, t=t)


def symmetric(bitmaps: Sequence, spec, r: int | None = None):
    """Arbitrary symmetric function ``spec.accept[count]`` (oracle.py:17-31)."""
    accept_bytes(spec, len(bitmaps))
    return _run(bitmaps, r, accept=spec)


def scan_count(bitmaps: Sequence, t: int, r: int | None = None, budget_bytes: int = DEFAULT_BUDGET_BYTES,
               stats: dict | None = None):
    """counters.scan_count (counters.py:46-67).

    ``budget_bytes`` keeps the reference's contract exactly (counters.py:54-57):
    r counters of counter_width(N) bits may not exceed it, else ResourceError
    with the reference's message, although the kernel keeps its counters in
    registers.  ``threshold`` is the same query without the budget."""
    _check_t(len(bitmaps), t)
    if r is None:
        r = max(b.bit_length for b in bitmaps)
    width = counter_width(len(bitmaps))
    if r * width // 8 > budget_bytes:
        raise ResourceError(
            f"{r} counters of {width} bits exceed the {budget_bytes}-byte budget; "
            "consider hash_count")
    res = _run(bitmaps, r, t=t)
    if stats is not None:
        stats["counter_width"] = counter_width(len(bitmaps))
        stats["increments"] = sum(_cardinality(b) for b in bitmaps)
    return res


def scan_count_symmetric(bitmaps: Sequence, spec, r: int | None = None):
    """counters.scan_count_symmetric (counters.py:70-83)."""
    acc = getattr(spec, "accept", spec)
    if len(acc) - 1 != len(bitmaps):
        raise InputError("spec arity does not match the input count")
    return _run(bitmaps, r, accept=spec)


def looped_threshold(bitmaps: Sequence, t: int, stats: dict | None = None):
    """circuits.looped_threshold (circuits/bitparallel.py:16-43)."""
    _check_t(len(bitmaps), t)
    res = _run(bitmaps, None, t=t)
    if stats is not None:
        stats["bitmap_ops"] = looped_op_count(len(bitmaps), t)
    return res


def csv_threshold(bitmaps: Sequence, t: int, stats: dict | None = None):
    """circuits.csv_threshold (circuits/bitparallel.py:51-129); requires 2 <= T < N (:63-64)."""
    n = len(bitmaps)
    if not 2 <= t < n:
        raise InputError(f"csv threshold needs 2 <= T < N, got T={t}, N={n}")
    res = _run(bitmaps, None, t=t)
    if stats is not None:
        stats["bitmap_ops"] = csv_op_count(n, t)
    return res


def _sweep_stats(bitmaps, t: int, stats: dict):
    """Fill ``stats`` with cdom's sweep counters, computed on the device (K8) from
    the cached query's directory; nothing for r = 0, like the reference (:209-210)."""
    r = max(b.bit_length for b in bitmaps)
    if word_count(r) == 0:
        return
    q = QUERIES.get(_classify(bitmaps), bitmaps, r, _device_for(bitmaps))
    stats.update(q.sweep_stats(t))


def cdom_threshold(bitmaps: Sequence, t: int, stats: dict | None = None):
    """runmerge.cdom_threshold (runmerge.py:198-241): RLE inputs only.  ``stats``
    receives what the reference's sweep reports (:237-240): segments, heap_pops
    and the dirty-segment dispatch counts under ``branches``, recomputed on the
    device (K8) -- except for T = 1 / T = N, which the reference answers with
    wide_or / wide_and without touching ``stats`` (:203-206)."""
    n = len(bitmaps)
    _check_t(n, t)
    if any(kind_of(b) not in ("r", "dr") for b in bitmaps):
        raise InputError("cdom operates on RLE bitmaps; compress inputs first")
    res = _run(bitmaps, None, t=t)
    if stats is not None and 1 < t < n:
        _sweep_stats(bitmaps, t, stats)
    return res


def cdom_symmetric(bitmaps: Sequence, spec, stats: dict | None = None):
    """runmerge.cdom_symmetric (runmerge.py:244-299): RLE inputs only.  ``stats``
    receives segments and heap_pops (:296-298), recomputed on the device (K8)."""
    accept_bytes(spec, len(bitmaps))
    if any(kind_of(b) not in ("r", "dr") for b in bitmaps):
        raise InputError("cdom operates on RLE bitmaps; compress inputs first")
    res = _run(bitmaps, None, accept=spec)
    if stats is not None:
        _sweep_stats(bitmaps, 0, stats)
    return res


SCANCOUNT_CUTOFF = 128  # runmerge.py:25


def dirty_segment_solver(blocks: Sequence[Sequence[int]], t_eff: int, force_branch: str | None = None,
                         scancount_cutoff: int = SCANCOUNT_CUTOFF, stats: dict | None = None) -> list:
    """runmerge.dirty_segment_solver (runmerge.py:59-126): per-word threshold over
    aligned blocks of dirty words, ``blocks[i][w]`` being input i's word at offset w.
    The dispatch (or / and / scan / looped, :69-83) is reproduced for ``stats`` and
    ``force_branch`` is validated as the reference does; every branch computes the
    same function, which is evaluated by the device's counting kernel (K1)."""
    nd = len(blocks)
    if not 1 <= t_eff <= nd:
        raise InputError(f"effective threshold {t_eff} outside [1, {nd}]")
    width = len(blocks[0])
    arr = np.array([list(b) for b in blocks], dtype=np.uint64).reshape(nd, width)
    branch = force_branch
    if branch is None:
        if t_eff == 1:
            branch = "or"
        elif t_eff == nd:
            branch = "and"
        elif t_eff >= scancount_cutoff:
            branch = "scan"
        else:
            beta = int(np.unpackbits(arr.view(np.uint8)).sum()) if arr.size else 0
            branch = "looped" if 2 * beta >= nd * t_eff else "scan"
    if stats is not None:
        stats[branch] = stats.get(branch, 0) + 1
    if branch not in ("or", "and", "looped", "scan"):
        raise InputError(f"unknown branch {force_branch!r}")
    if width == 0:
        return []
    device = torch.device("cuda", torch.cuda.current_device())
    pitch = (width + 1) & ~1  # rows 16-byte aligned (bq.h)
    padded = np.zeros((nd, pitch), dtype=np.uint64)
    padded[:, :width] = arr
    rows = torch.from_numpy(padded.view(np.int64)).to(device)
    q = ThresholdQuery([DeviceBitmap(rows[i], 64 * width, width) for i in range(nd)], 64 * width, device=device)
    try:
        out, _ = q.threshold(t_eff)
        return [int(w) for w in out[:width].cpu().numpy().view(np.uint64)]
    finally:
        q.close()


def wide_or(bitmaps: list):
    """bitmaps.wide_or (bitmaps.py:647-667)."""
    if not bitmaps:
        raise InputError("wide_or of an empty list")
    if len(bitmaps) == 1:
        return bitmaps[0]
    return _run(bitmaps, None, t=1)


def wide_and(bitmaps: list):
    """bitmaps.wide_and (bitmaps.py:670-677)."""
    if not bitmaps:
        raise InputError("wide_and of an empty list")
    if len(bitmaps) == 1:
        return bitmaps[0]
    return _run(bitmaps, None, t=len(bitmaps))


class CircuitLibrary:
    """circuits.CircuitLibrary (circuits/library.py:84-133).

    ``keys`` / ``plan`` / ``program`` / ``build_circuit`` and the on-disk program
    cache behave as the reference's (``circuits.py`` holds this package's own
    builders, BitProgram layout and BQP1 disk format).  ``threshold`` plans the
    query exactly as the reference does -- so a request outside the table raises
    ``NoCoveringCircuit`` (library.py:66-67) and a bad (N, T) ``InputError`` --
    and then evaluates theta_T of the real inputs with the counting kernel: the
    padded circuit computes theta_T(B, 1^(T-T'), 0^...) = theta_T'(B), so the pad
    bitmaps are never materialised.  ``program(n, t)`` gives the tabulated
    straight-line program, which ``execute`` runs on the GPU (NVRTC)."""

    def __init__(self, n_max: int = 64, builder: str = "sideways", cache_dir: str | None = None):
        from . import circuits as C

        if builder not in C.BUILDERS:
            raise InputError(f"unknown builder {builder!r}")
        self.n_max = n_max
        self.builder = builder
        self.cache_dir = cache_dir
        self._programs: dict = {}
        self._keys = [(n, t) for n in C.tabulation_levels(n_max) for t in range(1, n + 1)]

    def keys(self):
        return list(self._keys)

    def build_circuit(self, n: int, t: int):
        from . import circuits as C

        return C.optimize(C.BUILDERS[self.builder](n, t))

    def program(self, n: int, t: int):
        """The tabulated (n, t) BitProgram, from memory, the cache directory, or
        built and compiled (then written to the cache directory)."""
        from . import circuits as C

        key = (n, t)
        prog = self._programs.get(key)
        if prog is not None:
            return prog
        path = C.program_path(self.cache_dir, self.builder, n, t)
        if path and os.path.exists(path):
            with open(path, "rb") as fp:
                prog = C.loads_program(fp.read())
        else:
            prog = C.compile_circuit(self.build_circuit(n, t))
            if path:
                os.makedirs(os.path.dirname(path), exist_ok=True)
                with open(path, "wb") as fp:
                    fp.write(C.dumps_program(prog))
        self._programs[key] = prog
        return prog

    def plan(self, n_req: int, t_req: int):
        from . import circuits as C

        return C.plan_padding(n_req, t_req, self._keys)

    def threshold(self, inputs: Sequence, t: int):
        self.plan(len(inputs), t)  # the reference's contract: InputError / NoCoveringCircuit
        return _run(inputs, None, t=t)


def _sibling_class(obj, name, default):
    """The class called ``name`` from the module that defined type(obj) (reference or ours)."""
    import importlib
    try:
        return getattr(importlib.import_module(type(obj).__module__), name, default)
    except Exception:
        return default


def decompress(bitmap):
    """bitmaps.decompress (bitmaps.py:417-431), decoded on the device (theta(1) of one stream).

    Raises FormatError on a malformed stream.  Device input -> DeviceBitmap."""
    if kind_of(bitmap) not in ("r", "dr"):
        raise InputError("decompress needs an RLE bitmap")
    if kind_of(bitmap) == "dr":
        return _run([bitmap], None, t=1)
    words = _run([to_device(bitmap)], None, t=1).to_numpy()
    nz = np.flatnonzero(words)
    cls = _sibling_class(bitmap, "UncompressedBitmap", UncompressedBitmap)
    return cls(words[: nz[-1] + 1 if nz.size else 0].tolist(), bitmap.bit_length)


def compress(bitmap):
    """bitmaps.compress (bitmaps.py:407-414): canonical encoding, returns RleBitmap
    (the reference class if the input is a reference object).  Encoded on the
    device (K7, bq_rle_encode_device); only the stream comes back to the host.
    (``compress_words``, the host encoder, serves the bitmap-type constructors.)"""
    k = kind_of(bitmap)
    if k not in ("u", "du"):
        raise InputError("compress needs an uncompressed bitmap")
    b = to_device(bitmap)
    enc = encode_device(b.data[: b.n_words], b.bit_length)
    return _sibling_class(bitmap, "RleBitmap", RleBitmap)(enc.tolist(), bitmap.bit_length)


def to_device(bitmap, device=None):
    """Upload a host bitmap (either representation) and return its device form."""
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    k = kind_of(bitmap)
    if k in ("du", "dr"):
        return bitmap
    t = to_device_words(host_words(bitmap), device)
    if k == "u":
        return DeviceBitmap(t, bitmap.bit_length, t.numel())
    return DeviceRleBitmap(t, bitmap.bit_length, t.numel())


def _cardinality(b) -> int:
    if hasattr(b, "cardinality"):
        return int(b.cardinality())
    return 0


# ---------------------------------------------------------------------------
# straight-line BitPrograms (circuits/programs.py), JIT-compiled for the GPU

class CompiledProgram:
    """A reference BitProgram (programs.py:56-72) compiled to an sm_100a kernel
    with NVRTC (bq_program_compile).  Duck-typed: anything with ``arity``,
    ``n_slots``, ``result_slot`` and ``instructions`` [(op, dst, a, b)]."""

    def __init__(self, program):
        self._lib = _lib.load()
        self.arity = int(program.arity)
        self.n_slots = int(program.n_slots)
        self.result_slot = int(program.result_slot)
        ins = np.asarray([tuple(i) for i in program.instructions], dtype=np.int32).reshape(-1, 4)
        self._ins = np.ascontiguousarray(ins)
        h = ctypes.c_void_p()
        _lib.check(self._lib.bq_program_compile(self._ins.ctypes.data if ins.size else None, len(ins), self.arity,
                                                self.n_slots, self.result_slot, ctypes.byref(h)),
                   "bq_program_compile")
        self._h = h

    def source(self) -> str:
        """Generated CUDA source (the GPU analogue of emit_source, programs.py:332-352)."""
        n = ctypes.c_uint64(0)
        _lib.check(self._lib.bq_program_source(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _lib.check(self._lib.bq_program_source(self._h, buf, n.value, ctypes.byref(n)))
        return buf.value.decode()

    def run(self, query: ThresholdQuery, out, popcnt, last_nz, stream=None):
        from .engine import stream_handle
        _lib.check(self._lib.bq_program_execute(self._h, query._h, out.data_ptr(), popcnt.data_ptr(),
                                                last_nz.data_ptr() if last_nz is not None else None,
                                                stream_handle(stream, query.device)), "bq_program_execute")

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._lib.bq_program_destroy(self._h)
        except Exception:
            pass


_PROGRAM_CACHE: dict = {}


def compile_program(program) -> CompiledProgram:
    """Compile (once per distinct program) and cache."""
    key = (int(program.arity), int(program.n_slots), int(program.result_slot),
           tuple(tuple(int(x) for x in i) for i in program.instructions))
    got = _PROGRAM_CACHE.get(key)
    if got is None:
        got = _PROGRAM_CACHE[key] = CompiledProgram(program)
    return got


def _check_program_inputs(program, inputs):
    if len(inputs) != program.arity:  # programs.py:240-242
        raise InputError(f"program expects {program.arity} inputs, got {len(inputs)}")
    if len({type(b) for b in inputs}) > 1:  # programs.py:243-245
        raise InputError("program inputs must share one representation")


def execute(program, inputs: Sequence):
    """circuits.execute (programs.py:163-193) on the GPU: any straight-line
    program over either representation; result of type(inputs[0])."""
    _check_program_inputs(program, inputs)
    r = max(b.bit_length for b in inputs)
    device = _device_for(inputs)
    nw = word_count(r)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device=device)
    popcnt = torch.zeros(1, dtype=torch.int64, device=device)
    last_nz = torch.zeros(1, dtype=torch.int64, device=device)
    if kind_of(inputs[0]) in ("r", "dr"):  # decode RLE inputs on the device first
        decoded = []
        for d in _dev_inputs(inputs, device):
            rq = RleQuery([d], r, device=device)
            words, _ = rq.threshold(1)
            rq.close()
            decoded.append(DeviceBitmap(words[:nw], r, nw))
        q = ThresholdQuery(decoded, r, device=device)
    else:
        q = QUERIES.get("u", inputs, r, device)
    compile_program(program).run(q, out, popcnt, last_nz)
    return _finish(inputs, out, nw, r, popcnt, last_nz)


def execute_horizontal(program, inputs: Sequence, batch_words: int = 256):
    """circuits.execute_horizontal (programs.py:196-237): uncompressed inputs
    only.  The GPU evaluates every word column in parallel, so ``batch_words``
    (the reference's CPU tile) does not change the result and is ignored."""
    _check_program_inputs(program, inputs)
    if kind_of(inputs[0]) not in ("u", "du"):
        raise InputError("horizontal execution requires uncompressed bitmaps")
    return execute(program, inputs)


# ---------------------------------------------------------------------------
# whole-bitmap set algebra on the device (bitmaps.py:438-677)

_OPS = {"and": 0, "or": 1, "xor": 2, "andnot": 3}


def _operand_words(b, r, device):
    """Device words of an operand: uncompressed as is, RLE decoded on the device."""
    k = kind_of(b)
    if k == "du":
        return b.data, b.n_words
    if k == "u":
        t = UPLOADS.get(b, device)
        return t, t.numel()
    d = b if k == "dr" else DeviceRleBitmap(UPLOADS.get(b, device), b.bit_length)
    q = RleQuery([d], r, device=device)
    words, _ = q.threshold(1)
    q.close()
    return words, word_count(r)


def _set_op(kind: int, a, b, r: int):
    device = _device_for([a] if b is None else [a, b])
    ta, na = _operand_words(a, r, device)
    tb, nb = (None, 0) if b is None else _operand_words(b, r, device)
    nw = word_count(r)
    out = torch.empty(max(nw, 2), dtype=torch.int64, device=device)
    popcnt = torch.zeros(1, dtype=torch.int64, device=device)
    last_nz = torch.zeros(1, dtype=torch.int64, device=device)
    from .engine import stream_handle
    lib = _lib.load()
    _lib.check(lib.bq_binary_op(kind, ta.data_ptr() if na else None, na,
                                (tb.data_ptr() if nb else None) if tb is not None else None, nb, r,
                                out.data_ptr(), popcnt.data_ptr(), last_nz.data_ptr(),
                                stream_handle(None, device)), "bq_binary_op")
    return _finish([a], out, nw, r, popcnt, last_nz)


def _check_same_type(a, b):
    if type(a) is not type(b):  # bitmaps.py:591-595
        raise InputError("mixed bitmap representations; convert explicitly with compress/decompress")


def binary_op(kind: str, a, b):
    """bitmaps.binary_op (bitmaps.py:629-635) on the device."""
    try:
        code = _OPS[kind.lower()]
    except KeyError:
        raise InputError(f"unknown operation {kind!r}") from None
    _check_same_type(a, b)
    return _set_op(code, a, b, max(a.bit_length, b.bit_length))


def and_(a, b):
    return binary_op("and", a, b)


def or_(a, b):
    return binary_op("or", a, b)


def xor(a, b):
    return binary_op("xor", a, b)


def andnot(a, b):
    return binary_op("andnot", a, b)


def not_(a, bit_length: int):
    """bitmaps.not_ (bitmaps.py:638-644): complement within [0, bit_length)."""
    if bit_length < a.bit_length:
        raise InputError("complement universe smaller than the bitmap")
    return _set_op(4, a, None, bit_length)
