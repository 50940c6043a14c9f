"""BQBM serialization (reference bitmaps.py:689-732) against bytes and errors the
reference produced (tests/golden/serial.json, made by make_golden.serial_cases).
Header / payload / uncompressed-tail errors are raised before any device work
and run on CPU; loads to the device and RLE validation (K3) need the GPU."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

SERIAL = json.load(open(os.path.join(GOLDEN, "serial.json")))
HOST_ERRORS = {"truncated_header", "bad_magic", "truncated_payload", "unknown_tag", "u_bits_beyond_r",
               "u_too_many_words"}


def _host(case):
    from paper_1402_4073_b200 import RleBitmap, UncompressedBitmap

    cls = UncompressedBitmap if case["kind"] == "U" else RleBitmap
    return cls([int(w) for w in case["words"]], case["r"])


@pytest.mark.parametrize("case", SERIAL["valid"], ids=lambda c: f'{c["kind"]}{c["r"]}')
def test_writer_matches_reference_bytes(case):
    from paper_1402_4073_b200 import dumps_bitmap

    assert dumps_bitmap(_host(case)).hex() == case["hex"]


@pytest.mark.parametrize("case", [c for c in SERIAL["invalid"] if c["name"] in HOST_ERRORS], ids=lambda c: c["name"])
def test_reader_rejects_like_reference_before_upload(case):
    from paper_1402_4073_b200 import FormatError, loads_bitmap_device

    assert case["error"] == "FormatError"
    with pytest.raises(FormatError) as ei:
        loads_bitmap_device(bytes.fromhex(case["hex"]))
    assert str(ei.value) == case["message"]


def test_reader_handles_non_seekable_streams():
    from paper_1402_4073_b200 import FormatError
    from paper_1402_4073_b200.serial import read_bitmap_device

    class Pipe(io.RawIOBase):
        def __init__(self, data):
            self._b = io.BytesIO(data)

        def readable(self):
            return True

        def readinto(self, b):
            chunk = self._b.read(min(len(b), 7))  # short reads
            b[:len(chunk)] = chunk
            return len(chunk)

    case = next(c for c in SERIAL["invalid"] if c["name"] == "truncated_payload")
    with pytest.raises(FormatError, match="truncated bitmap payload"):
        read_bitmap_device(io.BufferedReader(Pipe(bytes.fromhex(case["hex"])), buffer_size=16))


# ---- device side -------------------------------------------------------------

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def _device_words(b):
    return [int(w) for w in b.data[: b.n_words].cpu().numpy().view(np.uint64)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SERIAL["valid"], ids=lambda c: f'{c["kind"]}{c["r"]}')
def test_load_to_device_and_back(bq, case, tmp_path):
    data = bytes.fromhex(case["hex"])
    b = bq.loads_bitmap_device(data)
    assert isinstance(b, bq.DeviceBitmap if case["kind"] == "U" else bq.DeviceRleBitmap)
    assert b.bit_length == case["r"] and _device_words(b) == [int(w) for w in case["words"]]
    assert bq.dumps_bitmap(b) == data
    path = tmp_path / "b.bqbm"
    with open(path, "wb") as fp:
        bq.write_bitmap(fp, b)
    with open(path, "rb") as fp:
        again = bq.read_bitmap_device(fp)
    assert _device_words(again) == [int(w) for w in case["words"]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SERIAL["invalid"], ids=lambda c: c["name"])
def test_reader_matches_reference_on_malformed_input(bq, case):
    data = bytes.fromhex(case["hex"])
    if case["error"] is None:
        b = bq.loads_bitmap_device(data)
        assert ("U" if isinstance(b, bq.DeviceBitmap) else "R") == case["kind"]
        assert b.bit_length == case["r"] and _device_words(b) == [int(w) for w in case["words"]]
        return
    assert case["error"] == "FormatError"
    with pytest.raises(bq.FormatError) as ei:
        bq.loads_bitmap_device(data)
    assert str(ei.value) == case["message"]


@pytest.mark.gpu
def test_loaded_rle_feeds_the_hot_path(bq):
    """A stream loaded straight to HBM is a valid cdom input (no host decode)."""
    from oracle import oracle as O

    valid = [c for c in SERIAL["valid"] if c["kind"] == "R" and c["r"] == 70001][0]
    b = bq.loads_bitmap_device(bytes.fromhex(valid["hex"]))
    res = bq.cdom_threshold([b, b, b], 2)
    exp = O.cdom_threshold([np.array([int(w) for w in valid["words"]], dtype=np.uint64)] * 3, 70001, 2)
    got = res.to_numpy()
    assert np.array_equal(got[: exp.size], exp) and not got[exp.size:].any()
