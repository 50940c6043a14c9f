"""Bitmap types: the reference's two host representations, mirrored, plus
their HBM-resident counterparts.

* :class:`UncompressedBitmap` / :class:`RleBitmap` keep the reference API
  (reference bitmaps.py:54-345): ``words`` is a ``list[int]`` of LSB-first
  64-bit words, ``bit_length`` is r, trailing zero words are trimmed at
  construction (:66-67), bits >= r are rejected (:70-72).  They exist so the
  package works without the reference installed; every entry point also
  accepts the reference's own objects (duck-typed on ``.words`` /
  ``.bit_length`` and the class name) and returns the caller's class.
* :class:`DeviceBitmap` / :class:`DeviceRleBitmap` hold the words in a CUDA
  tensor.  They are what the hot path consumes without marshalling; results
  of device inputs stay on the device.
"""

from __future__ import annotations

from typing import Iterable, Iterator

import numpy as np

from .errors import FormatError, InputError

W = 64
WORD_MASK = (1 << W) - 1


def word_count(bit_length: int) -> int:
    return (bit_length + W - 1) // W


def _iter_word_bits(word: int, base: int) -> Iterator[int]:
    while word:
        low = word & -word
        yield base + low.bit_length() - 1
        word ^= low


class UncompressedBitmap:
    """Set over [0, bit_length) as LSB-first 64-bit words (reference bitmaps.py:54-157)."""

    __slots__ = ("words", "bit_length", "_card")

    def __init__(self, words: list, bit_length: int):
        if bit_length < 0:
            raise InputError("bit_length must be nonnegative")
        while words and words[-1] == 0:
            words.pop()
        if len(words) > word_count(bit_length):
            raise InputError("more words than bit_length allows")
        if words and len(words) == word_count(bit_length) and bit_length % W:
            if words[-1] >> (bit_length % W):
                raise InputError("set bits at positions >= bit_length")
        self.words = words
        self.bit_length = bit_length
        self._card = None

    @classmethod
    def empty(cls, bit_length: int) -> "UncompressedBitmap":
        return cls([], bit_length)

    @classmethod
    def ones(cls, bit_length: int) -> "UncompressedBitmap":
        full, rem = divmod(bit_length, W)
        words = [WORD_MASK] * full
        if rem:
            words.append((1 << rem) - 1)
        return cls(words, bit_length)

    @classmethod
    def from_positions(cls, positions: Iterable[int], bit_length: int) -> "UncompressedBitmap":
        words = [0] * word_count(bit_length)
        prev = -1
        for p in positions:
            if p <= prev:
                raise InputError("positions must be strictly ascending")
            if p >= bit_length:
                raise InputError(f"position {p} out of range [0, {bit_length})")
            words[p >> 6] |= 1 << (p & 63)
            prev = p
        return cls(words, bit_length)

    def cardinality(self) -> int:
        if self._card is None:
            self._card = sum(w.bit_count() for w in self.words)
        return self._card

    def get(self, position: int) -> bool:
        if not 0 <= position < self.bit_length:
            raise InputError("position out of range")
        wi = position >> 6
        return wi < len(self.words) and bool(self.words[wi] >> (position & 63) & 1)

    __contains__ = get

    def iter_set_bits(self) -> Iterator[int]:
        for wi, word in enumerate(self.words):
            if word:
                yield from _iter_word_bits(word, wi << 6)

    def positions(self) -> list:
        return list(self.iter_set_bits())

    def __eq__(self, other):
        if not hasattr(other, "words") or type(other).__name__ != "UncompressedBitmap":
            return NotImplemented
        return self.bit_length == other.bit_length and list(self.words) == list(other.words)

    def __repr__(self):
        return f"UncompressedBitmap(card={self.cardinality()}, r={self.bit_length})"

    def iter_runs(self) -> Iterator[tuple]:
        """Maximal ``(start, end_inclusive, bit)`` runs covering [0, bit_length)
        (bitmaps.py:124-136), found word by word from bit transitions."""
        yield from _runs_from_words(self.words, self.bit_length)

    # set algebra (bitmaps.py:145-155) on the device: api.and_ / or_ / xor / andnot
    def __and__(self, other):
        from .api import and_
        return and_(self, other)

    def __or__(self, other):
        from .api import or_
        return or_(self, other)

    def __xor__(self, other):
        from .api import xor
        return xor(self, other)

    def andnot(self, other):
        from .api import andnot
        return andnot(self, other)


def _runs_from_words(words, r: int) -> Iterator[tuple]:
    """Runs of a word sequence (missing words zero) over [0, r): each word's bit
    transitions are located with bit tricks instead of a per-bit loop."""
    if r == 0:
        return
    start, prev = 0, words[0] & 1 if words else 0
    for wi in range(word_count(r)):
        w = words[wi] if wi < len(words) else 0
        base = wi * W
        nbits = min(W, r - base)
        # bit k of t is set where bit k differs from bit k-1 (bit -1 = the previous run's bit)
        t = (w ^ ((w << 1) | prev)) & ((1 << nbits) - 1)
        while t:
            k = (t & -t).bit_length() - 1
            yield start, base + k - 1, prev
            start, prev = base + k, prev ^ 1
            t &= t - 1
    yield start, r - 1, prev


class RleBitmap:
    """Word-aligned run-length encoding (reference bitmaps.py:160-345).

    Marker word: bit 0 fill bit, bits 1-32 fill run in words, bits 33-63 the
    number of literal words that follow (bitmaps.py:27-40)."""

    __slots__ = ("words", "bit_length", "_card")

    def __init__(self, words: list, bit_length: int):
        if bit_length < 0:
            raise InputError("bit_length must be nonnegative")
        self.words = words
        self.bit_length = bit_length
        self._card = None

    @classmethod
    def empty(cls, bit_length: int) -> "RleBitmap":
        words = []
        remaining = word_count(bit_length)
        while remaining:
            run = min(remaining, (1 << 32) - 1)
            words.append(run << 1)
            remaining -= run
        return cls(words, bit_length)

    @classmethod
    def from_words(cls, words, bit_length: int) -> "RleBitmap":
        from .api import compress_words
        return cls(compress_words(words, bit_length), bit_length)

    @classmethod
    def from_positions(cls, positions: Iterable[int], bit_length: int) -> "RleBitmap":
        return cls.from_words(UncompressedBitmap.from_positions(positions, bit_length).words, bit_length)

    @classmethod
    def ones(cls, bit_length: int) -> "RleBitmap":
        return cls.from_words(UncompressedBitmap.ones(bit_length).words, bit_length)

    def __eq__(self, other):
        if not hasattr(other, "words") or type(other).__name__ != "RleBitmap":
            return NotImplemented
        return self.bit_length == other.bit_length and list(self.words) == list(other.words)

    def __repr__(self):
        return f"RleBitmap(r={self.bit_length}, words={len(self.words)})"

    def iter_word_segments(self, total_words: int | None = None) -> Iterator[tuple]:
        """``('f', bit, count)`` fill and ``('d', start, count)`` literal segments,
        zero-extended to ``total_words`` (default: the bit length's word count);
        FormatError on a truncated literal group or coverage beyond it
        (bitmaps.py:196-219)."""
        words, n = self.words, len(self.words)
        i = covered = 0
        while i < n:
            mk = words[i]
            bit, run, dirty = mk & 1, (mk >> 1) & 0xFFFFFFFF, mk >> 33
            i += 1
            if run:
                yield "f", bit, run
                covered += run
            if dirty:
                if i + dirty > n:
                    raise FormatError("marker announces more literal words than present")
                yield "d", i, dirty
                i += dirty
                covered += dirty
        limit = word_count(self.bit_length) if total_words is None else total_words
        if covered > limit:
            raise FormatError("encoded words exceed bit_length")
        if covered < limit:
            yield "f", 0, limit - covered

    def _decoded_words(self) -> list:
        out = []
        for kind, a, b in self.iter_word_segments():
            out.extend([WORD_MASK if a else 0] * b if kind == "f" else self.words[a:a + b])
        return out

    def cardinality(self) -> int:
        if self._card is None:
            total = 0
            for kind, a, b in self.iter_word_segments():
                total += a * b * W if kind == "f" else sum(int(w).bit_count() for w in self.words[a:a + b])
            self._card = total
        return self._card

    def get(self, position: int) -> bool:
        if not 0 <= position < self.bit_length:
            raise InputError("position out of range")
        target, pos = position >> 6, 0
        for kind, a, b in self.iter_word_segments():
            if target < pos + b:
                return bool(a) if kind == "f" else bool(self.words[a + target - pos] >> (position & 63) & 1)
            pos += b
        return False

    __contains__ = get

    def iter_set_bits(self) -> Iterator[int]:
        pos = 0
        for kind, a, b in self.iter_word_segments():
            if kind == "f":
                if a:
                    yield from range(pos * W, (pos + b) * W)
            else:
                for k in range(b):
                    yield from _iter_word_bits(self.words[a + k], (pos + k) * W)
            pos += b

    def positions(self) -> list:
        return list(self.iter_set_bits())

    def iter_runs(self) -> Iterator[tuple]:
        """Maximal ``(start, end_inclusive, bit)`` runs over [0, bit_length) (bitmaps.py:221-259)."""
        yield from _runs_from_words(self._decoded_words(), self.bit_length)

    def run_count(self) -> int:
        return sum(1 for _ in self.iter_runs())

    def __and__(self, other):
        from .api import and_
        return and_(self, other)

    def __or__(self, other):
        from .api import or_
        return or_(self, other)

    def __xor__(self, other):
        from .api import xor
        return xor(self, other)

    def andnot(self, other):
        from .api import andnot
        return andnot(self, other)


class DeviceBitmap:
    """Uncompressed bitmap in HBM.

    ``data`` is a 1-D int64 CUDA tensor holding at least ``n_words`` words
    (bit patterns of uint64 words, LSB-first); words >= n_words read as zero.
    """

    __slots__ = ("data", "bit_length", "n_words", "_card")

    def __init__(self, data, bit_length: int, n_words: int | None = None, cardinality: int | None = None):
        if bit_length < 0:
            raise InputError("bit_length must be nonnegative")
        self.data = data
        self.bit_length = bit_length
        self.n_words = data.numel() if n_words is None else int(n_words)
        if self.n_words > word_count(bit_length):
            raise InputError("more words than bit_length allows")
        self._card = cardinality

    @property
    def device(self):
        return self.data.device

    def data_ptr(self) -> int:
        return self.data.data_ptr()

    def to_numpy(self) -> np.ndarray:
        return self.data[: self.n_words].cpu().numpy().view(np.uint64)

    def to_host(self, cls=UncompressedBitmap):
        words = self.to_numpy().tolist()
        return cls(words, self.bit_length)

    def cardinality(self) -> int:
        if self._card is None:
            self._card = int(np.unpackbits(self.to_numpy().view(np.uint8)).sum())
        return self._card

    def __repr__(self):
        return f"DeviceBitmap(r={self.bit_length}, words={self.n_words}, device={self.data.device})"


class DeviceRleBitmap:
    """RLE stream (reference marker format) in HBM: 1-D int64 CUDA tensor."""

    __slots__ = ("data", "bit_length", "n_words", "_span")

    def __init__(self, data, bit_length: int, n_words: int | None = None):
        self.data = data
        self.bit_length = bit_length
        self.n_words = data.numel() if n_words is None else int(n_words)
        self._span = None

    def data_ptr(self) -> int:
        return self.data.data_ptr()

    def span(self) -> tuple:
        """(device pointer or 0, stream words), computed once: streams are immutable
        (bitmaps.py:12-13), and a query over 1024 of them is ~1 ms of device work, so
        the per-stream torch attribute calls would show."""
        sp = self._span
        if sp is None:
            if not self.data.is_cuda:
                raise InputError("RLE streams must be CUDA tensors")
            sp = self._span = (self.data.data_ptr() if self.n_words else 0, self.n_words)
        return sp

    def to_host(self, cls=RleBitmap):
        return cls(self.data[: self.n_words].cpu().numpy().view(np.uint64).tolist(), self.bit_length)

    def __repr__(self):
        return f"DeviceRleBitmap(r={self.bit_length}, words={self.n_words})"


def kind_of(b) -> str:
    """'u' (uncompressed host), 'r' (RLE host), 'du' / 'dr' (device)."""
    if isinstance(b, DeviceBitmap):
        return "du"
    if isinstance(b, DeviceRleBitmap):
        return "dr"
    name = type(b).__name__
    if name == "UncompressedBitmap":
        return "u"
    if name == "RleBitmap":
        return "r"
    raise InputError(f"unsupported bitmap type {type(b).__name__}")
