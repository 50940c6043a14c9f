"""ctypes binding of libbq.so (include/bq.h).

The shared library is built in-tree (``paper_1402_4073_b200/libbq.so``, see
``csrc/Makefile`` / ``__graft_entry__.build``).  There is deliberately no CPU
fallback: if the library is missing every entry point raises
:class:`ExtensionMissing`.
"""

from __future__ import annotations

import ctypes

import numpy as np
import os
import threading

from .errors import DeviceError, ExtensionMissing, FormatError, InputError, ResourceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BQ_LIB", os.path.join(_HERE, "libbq.so"))

BQ_OK, BQ_EINPUT, BQ_ERESOURCE, BQ_EFORMAT, BQ_ECUDA = 0, -1, -2, -3, -4
BQ_MAX_INPUTS = 65535

_ERRORS = {BQ_EINPUT: InputError, BQ_ERESOURCE: ResourceError, BQ_EFORMAT: FormatError, BQ_ECUDA: DeviceError}


class Span(ctypes.Structure):
    _fields_ = [("words", ctypes.c_void_p), ("n_words", ctypes.c_uint64)]


_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I = ctypes.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "bq_version": (_I, []),
    "bq_last_error": (ctypes.c_char_p, []),
    "bq_release_cached_memory": (_I, []),
    "bq_query_create": (_I, [_P, _I, _U64, _U64, _U64, _I, _P]),
    "bq_query_destroy": (None, [_P]),
    "bq_query_out_words": (_U64, [_P]),
    "bq_query_threshold": (_I, [_P, _I, _P, _P, _P, _P]),
    "bq_query_symmetric": (_I, [_P, _P, _P, _P, _P, _P]),
    "bq_threshold_u64": (_I, [_P, _I, _U64, _I, _P, _P, _P]),
    "bq_symmetric_u64": (_I, [_P, _I, _U64, _P, _P, _P, _P]),
    "bq_shard_threshold": (_I, [_I, _P, _P, _I, _U64, _P, _P, _I, _P, _P, _P]),
    "bq_sweep_host": (_I, [_P, _P, _I, _U64, _P, _P, _I, _P, _P, _I, _U64]),
    "bq_release_workspace": (None, []),
    "bq_rle_query_create": (_I, [_P, _I, _U64, _I, _P]),
    "bq_rle_query_create_range": (_I, [_P, _I, _U64, _U64, _U64, _I, _P]),
    "bq_rle_query_destroy": (None, [_P]),
    "bq_rle_query_out_words": (_U64, [_P]),
    "bq_rle_query_directory_bytes": (_U64, [_P]),
    "bq_rle_query_layout_stats": (_I, [_P, _P, _P]),
    "bq_rle_query_layout_events": (_I, [_P, _P]),
    "bq_rle_query_sweep_stats": (_I, [_P, _I, _P, _P]),
    "bq_rle_query_threshold": (_I, [_P, _I, _P, _P, _P]),
    "bq_rle_query_symmetric": (_I, [_P, _P, _P, _P, _P]),
    "bq_rle_encode_host": (_I, [_P, _U64, _U64, _P, _U64, _P]),
    "bq_rle_encode_device": (_I, [_P, _U64, _U64, _P, _U64, _P, _P]),
    "bq_binary_op": (_I, [_I, _P, _U64, _P, _U64, _U64, _P, _P, _P, _P]),
    "bq_membership": (_I, [_P, _I, _P, _I, _P, _I]),
    "bq_rle_membership": (_I, [_P, _I, _P, _I, _P, _I]),
    "bq_program_compile": (_I, [_P, _I, _I, _I, _I, _P]),
    "bq_program_destroy": (None, [_P]),
    "bq_program_source": (_I, [_P, _P, _U64, _P]),
    "bq_program_execute": (_I, [_P, _P, _P, _P, _P, _P]),
    "bq_gen_bernoulli": (_I, [_U64, _U32, _U32, _U64, _U64, _P, _I, _P]),
    "bq_gen_bernoulli_rows": (_I, [_U64, _U32, _I, _P, _U64, _U64, _P, _U64, _P]),
    "bq_gen_density_q16": (_U32, [_U64, _U32, _U32, _U32]),
    "bq_gen_markov_rle": (_I, [_U64, _U32, _U64, ctypes.c_double, ctypes.c_double, _P, _U64, _P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libbq.so (once).  Raises ExtensionMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionMissing(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_1402_4073_b200/csrc`")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise ExtensionMissing(f"cannot load {LIB_PATH}: {exc}") from None
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str = ""):
    """Raise the reference-named exception for a libbq status code."""
    if rc == BQ_OK:
        return
    msg = load().bq_last_error().decode(errors="replace")
    cls = _ERRORS.get(rc, DeviceError)
    raise cls(f"{what}: {msg}" if what else msg)


def spans(pairs):
    """bq_span array (device_ptr, n_words) for the C ABI: a contiguous (n, 2) uint64
    numpy array (pass ``.ctypes.data``); built column-wise, no per-element ctypes."""
    arr = np.zeros((max(len(pairs), 1), 2), dtype=np.uint64)
    if pairs:
        arr[: len(pairs)] = np.asarray(pairs, dtype=np.uint64).reshape(-1, 2)
    return arr


def span_columns(ptrs, n_words):
    """The same from two sequences (pointers, word counts)."""
    arr = np.zeros((max(len(ptrs), 1), 2), dtype=np.uint64)
    if len(ptrs):
        arr[: len(ptrs), 0] = ptrs
        arr[: len(ptrs), 1] = n_words
    return arr
