"""Exception classes with the reference's names and bases (reference errors.py:4-25).

When the reference package ``bitquorum`` is importable, each class here also
derives from the reference class of the same name, so callers (and the
reference harness, which turns ``InputError``/``ResourceError`` into DNF at
bench/competitions.py:272-274) catch them unchanged.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from bitquorum import errors as _ref
except Exception:  # the reference is optional at run time
    _ref = None


def _bases(name, *fallback):
    if _ref is not None and hasattr(_ref, name):
        return (getattr(_ref, name),)
    return fallback


class BitquorumError(*_bases("BitquorumError", Exception)):
    """Base class for package errors."""


class InputError(*_bases("InputError", BitquorumError, ValueError)):
    """Caller supplied an argument outside an operation's contract."""


class FormatError(*_bases("FormatError", BitquorumError, ValueError)):
    """Serialized or encoded data is structurally invalid."""


class ResourceError(*_bases("ResourceError", BitquorumError, RuntimeError)):
    """An operation would exceed its configured memory or size budget."""


class CorrectnessError(*_bases("CorrectnessError", BitquorumError, RuntimeError)):
    """An algorithm produced output that disagrees with the reference result."""


class NoCoveringCircuit(*_bases("NoCoveringCircuit", BitquorumError, LookupError)):
    """No stored circuit can be padded to answer the requested query."""


class DeviceError(BitquorumError, RuntimeError):
    """A CUDA runtime failure inside libbq (no reference analogue)."""


class ExtensionMissing(BitquorumError, ImportError):
    """libbq.so was not built or cannot be loaded; there is no CPU fallback."""
