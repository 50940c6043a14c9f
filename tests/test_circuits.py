"""Host-side circuit construction (paper_1402_4073_b200/circuits.py): the
CircuitLibrary surface (keys / plan / program / build_circuit, the BQP1 program
cache) without the reference, and interoperability with the reference's own
programs and planner when it is importable.  CPU only."""

from __future__ import annotations

import itertools
import os
import sys

import pytest

from paper_1402_4073_b200 import circuits as C
from paper_1402_4073_b200.api import CircuitLibrary
from paper_1402_4073_b200.errors import InputError, NoCoveringCircuit, ResourceError

REF = os.environ.get("BQ_REFERENCE_SRC", "/root/reference/pkg/src")


def _ref():
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import bitquorum  # noqa: F401

    return bitquorum


@pytest.mark.parametrize("builder", sorted(C.BUILDERS))
def test_builders_compute_the_threshold_function(builder):
    for n in range(1, 10):
        for t in range(1, n + 1):
            c = C.optimize(C.BUILDERS[builder](n, t))
            for bits in itertools.product((0, 1), repeat=n):
                assert c.evaluate(bits) == int(sum(bits) >= t), (builder, n, t, bits)


def test_builder_contracts():
    with pytest.raises(InputError):
        C.build_sideways_sum(4, 5)
    with pytest.raises(InputError):
        C.build_tree_adder(0, 1)
    with pytest.raises(ResourceError):
        C.build_sop(40, 20)  # choose(40, 20) > SOP_TERM_CAP (core.py:259-263)


def test_program_format_round_trip_and_execution_semantics():
    for n, t in [(5, 2), (9, 9), (17, 6)]:
        prog = C.compile_circuit(C.optimize(C.build_sideways_sum(n, t)))
        assert C.loads_program(C.dumps_program(prog)) == prog
        assert prog.peak_slots <= prog.n_slots
        # interpret the program over all-bit-pattern "bitmaps" (one bit per input pattern)
        pats = list(itertools.product((0, 1), repeat=n))
        words = [sum(p[i] << k for k, p in enumerate(pats)) for i in range(n)]
        mask = (1 << len(pats)) - 1
        slots = words + [0] * (prog.n_slots - n)
        for op, d, a, b in prog.instructions:
            if op == C.OP_ZERO:
                slots[d] = 0
            elif op == C.OP_ONE:
                slots[d] = mask
            elif op == C.OP_AND:
                slots[d] = slots[a] & slots[b]
            elif op == C.OP_OR:
                slots[d] = slots[a] | slots[b]
            elif op == C.OP_XOR:
                slots[d] = slots[a] ^ slots[b]
            elif op == C.OP_ANDNOT:
                slots[d] = slots[a] & ~slots[b] & mask
            elif op == C.OP_NOT:
                slots[d] = ~slots[a] & mask
        res = slots[prog.result_slot]
        assert res == sum(int(sum(p) >= t) << k for k, p in enumerate(pats))


def test_padding_plan_kat_and_contract():
    # SPEC.md:551-552 / PAPER.md:1767-1771: request (10,7) against library {(16,8)}
    plan = C.plan_padding(10, 7, [(16, 8)])
    assert (plan.n, plan.t, plan.zero_pads, plan.one_pads) == (16, 8, 5, 1)
    plan = C.plan_padding(16, 8, [(16, 8)])
    assert (plan.zero_pads, plan.one_pads) == (0, 0)
    with pytest.raises(NoCoveringCircuit):
        C.plan_padding(10, 1, [(16, 8)])  # 1 not in [2, 8]
    lib = CircuitLibrary(n_max=16)
    plan = lib.plan(10, 7)  # the full table has (16, 7): zero pads only
    assert (plan.n, plan.t, plan.zero_pads, plan.one_pads) == (16, 7, 6, 0)
    with pytest.raises(NoCoveringCircuit):
        lib.plan(17, 3)
    with pytest.raises(NoCoveringCircuit):
        lib.threshold([object()] * 17, 3)  # planned before any device work (library.py:66-67)
    with pytest.raises(InputError):
        lib.plan(4, 5)
    assert (2, 1) in lib.keys() and (16, 16) in lib.keys() and all(n <= 16 for n, _ in lib.keys())


def test_program_cache_directory(tmp_path):
    lib = CircuitLibrary(n_max=8, builder="tree", cache_dir=str(tmp_path))
    p = lib.program(8, 3)
    path = tmp_path / "tree_n8_t3.bqp"
    assert path.exists()
    lib2 = CircuitLibrary(n_max=8, builder="tree", cache_dir=str(tmp_path))
    assert lib2.program(8, 3) == p


def test_plans_match_the_reference():
    ref = _ref()
    from bitquorum.circuits import library as RL

    keys = CircuitLibrary(n_max=64).keys()
    assert keys == RL.CircuitLibrary(n_max=64).keys()
    for n in range(1, 65):
        for t in range(1, n + 1):
            assert C.plan_padding(n, t, keys) == C.PaddingPlan(**vars(RL.plan_padding(n, t, keys)))
    del ref


def test_programs_interoperate_with_the_reference():
    """Our BQP1 bytes load in the reference and execute to the reference's own
    threshold answer; the reference's programs load here unchanged."""
    _ref()
    import random

    from bitquorum import bitmaps as bm
    from bitquorum import counters
    from bitquorum.circuits import programs as RP
    from bitquorum.circuits import core as RC

    rng = random.Random(3)
    for n, t in [(5, 2), (12, 7), (33, 17)]:
        ins = [bm.UncompressedBitmap([rng.getrandbits(64) for _ in range(20)], 64 * 20) for _ in range(n)]
        exp = counters.scan_count(ins, t)
        for builder in ("sideways", "tree", "sorter"):
            ours = C.compile_circuit(C.optimize(C.BUILDERS[builder](n, t)))
            assert RP.execute(RP.loads_program(C.dumps_program(ours)), ins) == exp
        theirs = RP.compile_circuit(RC.optimize(RC.build_sideways_sum(n, t)))
        back = C.loads_program(RP.dumps_program(theirs))
        assert RP.dumps_program(theirs) == C.dumps_program(back)
