"""BQBM bitmap files straight to and from HBM (reference bitmaps.py:689-732).

The reference format: header ``<4scQQ`` = magic ``b"BQBM"``, representation
tag (``b"U"`` uncompressed / ``b"R"`` RLE), bit_length, word count; then the
words as little-endian uint64.  The reference reader builds a Python list of
ints and, for RLE, validates by decompressing on the CPU (:702-722).  Here the
payload is read with ``readinto`` into a pinned host tensor and copied to the
device in one transfer; RLE streams are validated on the device by the K3
directory kernel (the same checks ``iter_word_segments`` makes), and
uncompressed payloads get the reference constructor's checks (trailing zero
words trimmed, nothing at or beyond bit_length, :63-73) on the pinned buffer
before the copy.  Errors and messages follow the reference reader.
"""

from __future__ import annotations

import io
import os
import re
import struct

import numpy as np

from .bitmaps import DeviceBitmap, DeviceRleBitmap, kind_of, word_count
from .errors import FormatError

MAGIC = b"BQBM"
_HEADER = struct.Struct("<4scQQ")
_TAGS = {"u": b"U", "du": b"U", "r": b"R", "dr": b"R"}


def _torch():
    import torch

    return torch


def _remaining(fp):
    try:
        if not fp.seekable():
            return None
        pos = fp.tell()
        end = fp.seek(0, os.SEEK_END)
        fp.seek(pos)
        return end - pos
    except (AttributeError, OSError, ValueError):
        return None


def _read_payload(fp, count: int):
    """``count`` words into a pinned int64 tensor, or FormatError when the file is shorter."""
    torch = _torch()
    nbytes = 8 * count
    rem = _remaining(fp)
    if rem is not None and rem < nbytes:
        fp.seek(0, os.SEEK_END)
        raise FormatError("truncated bitmap payload")
    host = torch.empty(count, dtype=torch.int64, pin_memory=torch.cuda.is_available())
    view = memoryview(host.numpy()).cast("B")
    got = 0
    readinto = getattr(fp, "readinto", None)
    while got < nbytes:
        if readinto is not None:
            k = readinto(view[got:])
        else:
            chunk = fp.read(nbytes - got)
            k = len(chunk)
            view[got:got + k] = chunk
        if not k:
            break
        got += k
    if got != nbytes:
        raise FormatError("truncated bitmap payload")
    return host


def _check_uncompressed(words: np.ndarray, bit_length: int) -> int:
    """The reference constructor's checks (bitmaps.py:63-73): trim trailing zero
    words, then reject words or bits beyond bit_length; returns the trimmed count."""
    nz = words != 0
    n = words.size - int(np.argmax(nz[::-1])) if nz.any() else 0
    nw = word_count(bit_length)
    if n > nw:
        raise FormatError("more words than bit_length allows")
    if n == nw and n and bit_length % 64 and int(words[n - 1]) >> (bit_length % 64):
        raise FormatError("set bits at positions >= bit_length")
    return n


def read_bitmap_device(fp, device=None):
    """``bitmaps.read_bitmap`` (bitmaps.py:702-722) producing a device bitmap:
    :class:`DeviceBitmap` for tag ``U``, :class:`DeviceRleBitmap` for ``R``."""
    torch = _torch()
    from .engine import RleQuery

    head = fp.read(_HEADER.size)
    if len(head) != _HEADER.size:
        raise FormatError("truncated bitmap header")
    magic, tag, bit_length, count = _HEADER.unpack(head)
    if magic != MAGIC:
        raise FormatError("bad bitmap magic")
    host = _read_payload(fp, count)
    if tag not in (b"U", b"R"):
        raise FormatError(f"unknown representation tag {tag!r}")
    n = _check_uncompressed(host.numpy().view(np.uint64), bit_length) if tag == b"U" else count
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if tag == b"U":
        data = host[:max(n, 1)].to(dev, non_blocking=True) if n else torch.zeros(1, dtype=torch.int64, device=dev)
        return DeviceBitmap(data, bit_length, n)
    data = host.to(dev, non_blocking=True) if count else torch.zeros(1, dtype=torch.int64, device=dev)
    bm = DeviceRleBitmap(data, bit_length, count)
    torch.cuda.current_stream(dev).synchronize()  # the K3 launch below runs on the legacy stream
    try:
        RleQuery([bm], bit_length)  # K3 walks the markers: the reference's decompress() validation
    except FormatError as exc:
        raise FormatError(re.sub(r"^.*?stream \d+: ", "", str(exc))) from None  # the reference's bare message
    return bm


def loads_bitmap_device(data: bytes, device=None):
    """``bitmaps.loads_bitmap`` (bitmaps.py:731-732) to the device."""
    return read_bitmap_device(io.BytesIO(data), device)


def _words_for_write(bitmap) -> tuple[bytes, np.ndarray]:
    from .engine import host_words

    k = kind_of(bitmap)
    if k == "du":
        w = bitmap.to_numpy()
        nz = np.flatnonzero(w)
        w = w[: int(nz[-1]) + 1 if nz.size else 0]  # the reference's words are trimmed
    elif k == "dr":
        w = bitmap.data[: bitmap.n_words].cpu().numpy().view(np.uint64)
    else:
        w = host_words(bitmap)
    return _TAGS[k], np.ascontiguousarray(w, dtype="<u8")


def write_bitmap(fp, bitmap) -> None:
    """``bitmaps.write_bitmap`` (bitmaps.py:697-699) for host or device bitmaps."""
    tag, w = _words_for_write(bitmap)
    fp.write(_HEADER.pack(MAGIC, tag, bitmap.bit_length, w.size))
    fp.write(w.tobytes())


def dumps_bitmap(bitmap) -> bytes:
    """``bitmaps.dumps_bitmap`` (bitmaps.py:725-728) for host or device bitmaps."""
    buf = io.BytesIO()
    write_bitmap(buf, bitmap)
    return buf.getvalue()
