"""The reference's own harness and bitmap objects driving the GPU path, on the
GPU box.  The reference (installed into oracle/_ref by build(); no
/root/reference there) supplies the datasets, the similarity queries and
run_competitions, which checks every algorithm against brute_threshold before
timing it (bench/competitions.py:237-309).  ``registry.register()`` adds ``gpu``
and ``gpu_cdom`` to its ALGORITHMS; every drop-in entry point is then called
with reference UncompressedBitmap / RleBitmap objects and compared with the
reference's own answer.  Needs a B200."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
bitquorum = pytest.importorskip("bitquorum", reason="reference not installed (oracle/install_ref.sh)")


@pytest.fixture(scope="module")
def bq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_4073_b200 as bq

    bq._lib.load()
    return bq


@pytest.fixture(scope="module")
def datasets():
    from bitquorum.bench.datagen import SyntheticSpec, gen_synthetic

    return [gen_synthetic(SyntheticSpec("uniform", 3, 400, 20000, 40)),
            gen_synthetic(SyntheticSpec("clustered", 5, 900, 50000, 40))]


@pytest.mark.parametrize("repr_kind", ["uncompressed", "ewah"])
def test_run_competitions_verifies_and_times_gpu(bq, datasets, repr_kind):
    from bitquorum.bench import competitions as comp

    from paper_1402_4073_b200 import registry

    names = registry.register(comp)
    assert set(names) <= set(comp.ALGORITHMS)
    algos = ["scancount", "looped", "gpu"] + (["cdom", "gpu_cdom"] if repr_kind == "ewah" else [])
    pairs = [(8, 3), (16, 1), (16, 16), (33, 7)]
    rows = comp.run_competitions(datasets, pairs, algo_names=algos, repr_kind=repr_kind, verify_only=True)
    verified = {(r.algorithm, r.n, r.t) for r in rows if r.flags == "verified"}
    for n, t in pairs:
        assert ("gpu", n, t) in verified
        if repr_kind == "ewah":
            assert ("gpu_cdom", n, t) in verified
    rows = comp.run_competitions(datasets[:1], [(16, 5)], algo_names=algos, repr_kind=repr_kind,
                                 min_total_ms=20.0)
    gpu = [r for r in rows if r.algorithm == "gpu"]
    assert gpu and gpu[0].ms_per_exec > 0 and gpu[0].rank >= 0


def test_drop_in_entry_points_with_reference_objects(bq, datasets):
    """Each entry point, given the reference's objects, returns what the
    reference's own function returns (same class, same words)."""
    from bitquorum import bitmaps as bm
    from bitquorum import counters, oracle, runmerge
    from bitquorum.circuits import CircuitLibrary, compile_circuit, csv_threshold, execute, looped_threshold
    from bitquorum.circuits import build_sideways_sum, optimize
    from bitquorum.circuits import execute_horizontal

    ds = datasets[1]
    u = ds.to_repr("uncompressed").bitmaps[:24]
    c = ds.to_repr("ewah").bitmaps[:24]
    spec = oracle.SymmetricSpec.interval(24, 2, 5)
    checks = [
        (bq.scan_count(u, 3), counters.scan_count(u, 3)),
        (bq.scan_count(c, 3), counters.scan_count(c, 3)),
        (bq.scan_count_symmetric(u, spec), counters.scan_count_symmetric(u, spec)),
        (bq.looped_threshold(u, 4), looped_threshold(u, 4)),
        (bq.csv_threshold(u, 5), csv_threshold(u, 5)),
        (bq.wide_or(u), bm.wide_or(u)),
        (bq.wide_and(u[:3]), bm.wide_and(u[:3])),
        (bq.wide_or(c), bm.wide_or(c)),
        (bq.cdom_threshold(c, 2), runmerge.cdom_threshold(c, 2)),
        (bq.cdom_symmetric(c, spec), runmerge.cdom_symmetric(c, spec)),
        (bq.CircuitLibrary(n_max=32).threshold(u, 6), CircuitLibrary(n_max=32).threshold(u, 6)),
        (bq.compress(u[0]), bm.compress(u[0])),
        (bq.decompress(c[1]), bm.decompress(c[1])),
        (bq.and_(u[0], u[1]), bm.and_(u[0], u[1])),
        (bq.or_(c[0], c[1]), bm.or_(c[0], c[1])),
        (bq.xor(u[2], u[3]), bm.xor(u[2], u[3])),
        (bq.andnot(c[2], c[3]), bm.andnot(c[2], c[3])),
        (bq.not_(u[4], u[4].bit_length + 70), bm.not_(u[4], u[4].bit_length + 70)),
    ]
    prog = compile_circuit(optimize(build_sideways_sum(24, 7)))
    checks.append((bq.execute(prog, u), execute(prog, u)))
    checks.append((bq.execute_horizontal(prog, u), execute_horizontal(prog, u)))
    checks.append((bq.execute(bq.CircuitLibrary(n_max=32).program(24, 7), u), counters.scan_count(u, 7)))
    for k, (got, exp) in enumerate(checks):
        assert type(got) is type(exp), k
        assert got == exp, k
    from bitquorum.errors import InputError, NoCoveringCircuit

    with pytest.raises(NoCoveringCircuit):
        bq.CircuitLibrary(n_max=16).threshold(u, 3)
    with pytest.raises(InputError):  # the harness's DNF class (competitions.py:272-274)
        bq.csv_threshold(u, 24)


@pytest.mark.parametrize("seed", range(6))
def test_dirty_segment_solver_every_branch(bq, seed):
    """runmerge.dirty_segment_solver (runmerge.py:59-126): the dispatch counts and
    the words, with each branch forced (SPEC's cross-branch equality) and unforced,
    against the reference's own solver on the same blocks."""
    import random

    from bitquorum import runmerge

    rng = random.Random(seed)
    nd = rng.choice([1, 2, 5, 40, 130, 200])
    width = rng.choice([1, 3, 17, 64])
    dens = rng.choice([0.02, 0.5, 0.95])
    blocks = [[sum(1 << b for b in range(64) if rng.random() < dens) for _ in range(width)] for _ in range(nd)]
    for t in sorted({1, nd, max(1, nd // 3), min(nd, 129)}):
        exp_st, got_st = {}, {}
        exp = runmerge.dirty_segment_solver(blocks, t, stats=exp_st)
        assert bq.dirty_segment_solver(blocks, t, stats=got_st) == exp
        assert got_st == exp_st
        for br in ("or", "and", "scan", "looped"):
            # forced branches only compute the threshold when they apply (OR: T=1, AND: T=nd)
            if (br == "or" and t != 1) or (br == "and" and t != nd):
                continue
            assert bq.dirty_segment_solver(blocks, t, force_branch=br) == exp
    with pytest.raises(bq.InputError):
        bq.dirty_segment_solver(blocks, nd + 1)
    with pytest.raises(bq.InputError):
        bq.dirty_segment_solver(blocks, 1, force_branch="heap")
