"""Shared fixtures: golden-case loading and the ``gpu`` marker."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# The Python reference installed by build() (oracle/install_ref.sh) -- present in
# the build container and, through the gpurun snapshot, on the GPU box.  Put on
# the path before the package is imported, so the package's exception classes
# derive from the reference's (errors.py) as they do in a reference install.
REF_INSTALL = os.path.join(ROOT, "oracle", "_ref")
if os.path.isdir(os.path.join(REF_INSTALL, "bitquorum")) and REF_INSTALL not in sys.path:
    sys.path.append(REF_INSTALL)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


class GoldenCase:
    """One reference-generated case: inputs (word arrays), bit lengths, expected words."""

    def __init__(self, arrays, prefix):
        flat = arrays[prefix + "in"]
        off = arrays[prefix + "off"].astype(np.int64)
        self.inputs = [flat[off[i]:off[i + 1]].copy() for i in range(len(off) - 1)]
        self.bits = [int(b) for b in arrays[prefix + "bits"]]
        self.out = arrays[prefix + "out"].copy()
        self.meta = json.loads(str(arrays[prefix + "meta"]))
        self.id = prefix.rstrip("_")

    @property
    def r(self):
        return int(self.meta["r"])

    @property
    def n(self):
        return len(self.inputs)


def load_golden(name):
    arrays = np.load(os.path.join(GOLDEN, name + ".npz"))
    prefixes = sorted({k.split("_")[0] + "_" for k in arrays.files})
    return [GoldenCase(arrays, p) for p in prefixes]


def load_kat():
    with open(os.path.join(GOLDEN, "kat.json")) as fp:
        return json.load(fp)


def padded(words, r):
    """Expected result words padded back to word_count(r) (the reference trims)."""
    out = np.zeros((r + 63) // 64, dtype=np.uint64)
    out[: len(words)] = words
    return out
