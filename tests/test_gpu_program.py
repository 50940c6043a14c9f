"""The reference's straight-line BitPrograms (TreeAdd, SSum, SrtCkt, SoP,
build_symmetric) JIT-compiled with NVRTC and run on the B200, against the
reference's own execute() results (tests/golden/programs.npz)."""

from __future__ import annotations

import types

import numpy as np
import pytest

from conftest import load_golden, padded
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PROGS = load_golden("programs")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


def as_program(meta):
    return types.SimpleNamespace(arity=meta["arity"], n_slots=meta["n_slots"], result_slot=meta["result_slot"],
                                 peak_slots=meta["peak_slots"], instructions=[tuple(i) for i in meta["instructions"]])


@pytest.mark.parametrize("case", PROGS, ids=lambda c: c.meta["label"])
def test_program_matches_reference_execute(bq, case):
    prog = as_program(case.meta)
    ins = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    got = bq.execute(prog, ins)
    assert got.words == case.out.tolist()
    assert got.bit_length == case.r
    assert got.cardinality() == case.meta["card"]
    assert bq.execute_horizontal(prog, ins).words == case.out.tolist()
    # RLE inputs -> canonical RLE result, as the reference's execute returns
    rle = [bq.compress(b) for b in ins]
    got_rle = bq.execute(prog, rle)
    assert isinstance(got_rle, bq.RleBitmap)
    assert [str(w) for w in got_rle.words] == case.meta["rle_out"]


def test_program_errors_and_source(bq):
    case = PROGS[0]
    prog = as_program(case.meta)
    ins = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    with pytest.raises(bq.InputError):
        bq.execute(prog, ins[:-1])
    with pytest.raises(bq.InputError):
        bq.execute_horizontal(prog, [bq.compress(b) for b in ins])
    src = bq.compile_program(prog).source()
    assert "bq_prog" in src and f"arity={prog.arity}" in src


def test_large_program_vs_counting_kernel(bq):
    """SSum(64, 32) program shape: the JIT'd program and the counting kernel agree
    on 2^16 words of generator data."""
    case = next(c for c in PROGS if c.meta["label"] == "tree(64,32)")
    prog = as_program(case.meta)
    lib = bq._lib.load()
    nw = 1 << 16
    arrs = []
    for i in range(64):
        a = np.empty(nw, dtype=np.uint64)
        lib.bq_gen_bernoulli(7, i, 32768, 0, nw, a.ctypes.data, 0, None)
        arrs.append(a)
    dev = [bq.DeviceBitmap(torch.from_numpy(a.view(np.int64)).cuda(), 64 * nw) for a in arrs]
    got = bq.execute(prog, dev)
    exp = O.threshold_port(arrs, 64 * nw, 32)
    assert np.array_equal(got.to_numpy(), exp)


SIM = load_golden("similarity")


@pytest.mark.parametrize("case", SIM, ids=lambda c: c.id)
def test_similarity_front_end_matches_reference(bq, case):
    """make_similarity (bench/similarity.py:26-58) with device membership, both
    representations, then the threshold over the replicated inputs."""
    from paper_1402_4073_b200.similarity import make_similarity

    m = case.meta
    for rle in (False, True):
        if rle:
            bms = [bq.compress(bq.UncompressedBitmap(a.tolist(), b)) for a, b in zip(case.inputs, case.bits)]
        else:
            bms = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
        ds = types.SimpleNamespace(name=m["name"], universe=m["universe"], bitmaps=bms)
        q = make_similarity(ds, m["rid_count"], m["n"], m["seed"])
        assert q.rids == m["rids"] and q.source_indices == m["chosen"] and q.multiplicities == m["mult"]
        got = bq.scan_count(q.bitmaps, m["t"])
        words = bq.decompress(got).words if rle else got.words
        assert words == case.out.tolist()


@pytest.mark.parametrize("case", SIM[:4], ids=lambda c: c.id)
def test_device_dataset_matches_reference_selection(bq, case):
    """DeviceDataset (datagen.Dataset in HBM): both representations produced on the
    device give the reference's selection and threshold answer."""
    from oracle import oracle as O
    from paper_1402_4073_b200.similarity import DeviceDataset, make_similarity

    m = case.meta
    host = [bq.UncompressedBitmap(a.tolist(), b) for a, b in zip(case.inputs, case.bits)]
    ds = types.SimpleNamespace(name=m["name"], universe=m["universe"], bitmaps=host)
    for kind in ("uncompressed", "ewah"):
        dd = DeviceDataset.from_dataset(ds, kind)
        assert len(dd.labels) == len(host)
        if kind == "ewah":
            for b, h in zip(dd.bitmaps, host):
                exp = O.rle_compress(np.array(h.words, dtype=np.uint64), h.bit_length)
                assert b.data[: b.n_words].cpu().numpy().view(np.uint64).tolist() == list(exp)
        q = make_similarity(dd, m["rid_count"], m["n"], m["seed"])
        assert q.rids == m["rids"] and q.source_indices == m["chosen"] and q.multiplicities == m["mult"]
        got = bq.scan_count(q.bitmaps, m["t"])  # device inputs of either kind: uncompressed device result
        assert isinstance(got, bq.DeviceBitmap)
        words = got.to_numpy()
        nz = np.flatnonzero(words)
        assert words[: nz[-1] + 1 if nz.size else 0].tolist() == case.out.tolist()
    assert dd.compressed_words() == sum(len(bq.compress(h).words) for h in host)
    with pytest.raises(bq.InputError):
        dd.to_repr("roaring")
