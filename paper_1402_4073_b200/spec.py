"""SymmetricSpec with the reference's constructors (reference oracle.py:17-53).

Entry points accept either this class, the reference's own ``SymmetricSpec``,
or a plain sequence of booleans (anything with ``.accept`` or iterable)."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InputError


@dataclass(frozen=True)
class SymmetricSpec:
    """``accept[k]`` is the output when exactly k of the inputs are 1."""

    accept: tuple

    def __post_init__(self):
        if len(self.accept) < 1:
            raise InputError("accept vector must have length arity + 1")

    @property
    def arity(self) -> int:
        return len(self.accept) - 1

    @classmethod
    def threshold(cls, n: int, t: int) -> "SymmetricSpec":
        if not 1 <= t <= n:
            raise InputError(f"threshold {t} outside [1, {n}]")
        return cls(tuple(k >= t for k in range(n + 1)))

    @classmethod
    def delta(cls, n: int, t: int) -> "SymmetricSpec":
        if not 0 <= t <= n:
            raise InputError(f"delta point {t} outside [0, {n}]")
        return cls(tuple(k == t for k in range(n + 1)))

    @classmethod
    def interval(cls, n: int, lo: int, hi: int) -> "SymmetricSpec":
        return cls(tuple(lo <= k <= hi for k in range(n + 1)))

    @classmethod
    def parity(cls, n: int) -> "SymmetricSpec":
        return cls(tuple(k % 2 == 1 for k in range(n + 1)))
