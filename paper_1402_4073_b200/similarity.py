"""Similarity-query construction, the hot path's caller in the paper's workload
(reference bench/similarity.py:26-58).

``make_similarity`` picks prototype row ids with the reference's seeded RNG,
keeps the dataset bitmaps that contain any of them, and truncates or
replicates them to exactly ``n`` inputs.  The (bitmaps x rids) membership
matrix is computed on the GPU in one kernel (``bq_membership`` /
``bq_rle_membership``) instead of one Python ``get`` per pair; replicated inputs
are the same objects repeated, so the query's device pointer table repeats
pointers and no bitmap is copied.
"""

from __future__ import annotations

import ctypes
import random
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .api import _device_for, compress_device, decompress, to_device
from .bitmaps import DeviceBitmap, DeviceRleBitmap, kind_of
from .engine import UPLOADS
from .errors import InputError


@dataclass
class DeviceDataset:
    """``bench.datagen.Dataset`` (datagen.py:29-56) with its bitmaps in HBM: a named
    collection over a shared universe of row ids.  ``make_similarity`` accepts it
    like the reference's dataset; representation changes run on the device
    (K7 encoder for ``ewah``, the K4 decoder for ``uncompressed``)."""

    name: str
    universe: int
    bitmaps: list
    labels: list = field(default_factory=list)

    def __post_init__(self):
        if not self.labels:
            self.labels = [str(i) for i in range(len(self.bitmaps))]

    @classmethod
    def from_dataset(cls, dataset, kind: str | None = None, device=None) -> "DeviceDataset":
        """Upload a (reference or host) dataset; each distinct bitmap object is copied once."""
        seen = {}
        bms = []
        for b in dataset.bitmaps:
            if id(b) not in seen:
                seen[id(b)] = to_device(b, device)
            bms.append(seen[id(b)])
        out = cls(dataset.name, dataset.universe, bms, list(getattr(dataset, "labels", []) or []))
        return out.to_repr(kind) if kind else out

    def to_repr(self, kind: str) -> "DeviceDataset":
        """Dataset.to_repr (datagen.py:42-52) on the device."""
        if kind in ("ewah", "rle", "compressed"):
            conv = [compress_device(b) for b in self.bitmaps]
        elif kind in ("uncompressed", "bitset"):
            conv = [b if isinstance(b, DeviceBitmap) else decompress(b) for b in self.bitmaps]
        else:
            raise InputError(f"unknown representation {kind!r}")
        return DeviceDataset(self.name, self.universe, conv, list(self.labels))

    def compressed_words(self) -> int:
        """Dataset.compressed_words (datagen.py:54-56)."""
        return sum(b.n_words if isinstance(b, DeviceRleBitmap) else compress_device(b).n_words for b in self.bitmaps)


@dataclass
class SimilarityQuery:
    dataset: str
    rids: list
    n: int
    source_indices: list
    multiplicities: list
    bitmaps: list

    def __post_init__(self):
        assert len(self.bitmaps) == self.n


def membership(bitmaps, rids, device=None) -> np.ndarray:
    """bool matrix [len(bitmaps), len(rids)]: bit rid of each bitmap (get(), bitmaps.py:107-113, :314-325)."""
    kinds = {kind_of(b) for b in bitmaps}
    rle = bool(kinds & {"r", "dr"})
    if rle and not kinds <= {"r", "dr"}:
        raise InputError("mixed bitmap representations; convert explicitly with compress/decompress")
    device = device if device is not None else _device_for(bitmaps)
    spans = (_lib.Span * max(len(bitmaps), 1))()
    keep = []
    for k, b in enumerate(bitmaps):
        if isinstance(b, (DeviceBitmap, DeviceRleBitmap)):
            t, nw = b.data, b.n_words
        else:
            t = UPLOADS.get(b, device)
            nw = t.numel()
        keep.append(t)
        spans[k].words = t.data_ptr() if nw else None
        spans[k].n_words = nw
    order = np.argsort(np.asarray(rids, dtype=np.uint64), kind="stable")
    srt = np.ascontiguousarray(np.asarray(rids, dtype=np.uint64)[order])
    out = np.zeros((len(bitmaps), len(rids)), dtype=np.uint8)
    if len(bitmaps) and len(rids):
        lib = _lib.load()
        fn = lib.bq_rle_membership if rle else lib.bq_membership
        _lib.check(fn(spans, len(bitmaps), srt.ctypes.data, len(rids), out.ctypes.data, device.index), "membership")
    res = np.empty_like(out)
    res[:, order] = out
    return res.astype(bool)


def make_similarity(dataset, rid_count: int, n: int, seed: int, max_retries: int = 64) -> SimilarityQuery:
    """bench.similarity.make_similarity (similarity.py:26-58): same seeds, same
    selection, same replication rule; ``dataset`` needs ``name``, ``universe``
    and ``bitmaps`` (the reference's Dataset qualifies)."""
    if not dataset.bitmaps:
        raise InputError("empty dataset")
    rows = dataset.universe
    rid_count = min(rid_count, rows)
    bitmaps = list(dataset.bitmaps)
    for attempt in range(max_retries):
        rng = random.Random(f"sim;{dataset.name};{rid_count};{n};{seed};{attempt}")
        rids = sorted(rng.sample(range(rows), rid_count))
        member = membership(bitmaps, rids)
        selected = []
        for i, b in enumerate(bitmaps):
            # any(b.get(rid) for rid in rids): get() raises for rid >= bit_length, short-circuit on a hit
            for j, rid in enumerate(rids):
                if not 0 <= rid < b.bit_length:
                    raise InputError("position out of range")
                if member[i, j]:
                    selected.append(i)
                    break
        if not selected:
            continue
        if len(selected) >= n:
            chosen = selected[:n]
            multiplicities = [1] * n
        else:
            chosen = selected
            base, extra = divmod(n, len(selected))
            multiplicities = [base + 1 if i < extra else base for i in range(len(selected))]
        resolved = []
        for idx, mult in zip(chosen, multiplicities):
            resolved.extend([bitmaps[idx]] * mult)
        return SimilarityQuery(dataset.name, rids, n, chosen, multiplicities, resolved)
    raise InputError(f"no bitmap contains any prototype rid after {max_retries} seeds")
