"""Threshold circuits and straight-line BitPrograms, host side.

Mirrors the construction API of the reference's ``circuits`` package
(``circuits/core.py``, ``programs.py``, ``library.py``) so that
``CircuitLibrary.plan`` / ``program`` / ``build_circuit`` and the on-disk
program cache work without the reference installed.  None of this is on the
device hot path: a threshold query runs the bit-sliced counting kernel (K1) and
any BitProgram runs as one NVRTC-compiled kernel (``api.execute``).  The
constructions here are this package's own (a gate builder that folds constants
and shares identical gates as it goes); they compute the same functions as the
reference's builders, so results agree bit for bit, but gate counts can differ
(the paper's counts are reproduced by the reference, not here).

Node and opcode conventions follow the reference so that programs interoperate:
nodes are ``(kind, a, b)`` with kinds ``input/const0/const1/and/or/xor/andnot/
not`` (core.py:23-30); programs are ``(opcode, dst, a, b)`` with opcodes 0..7
(programs.py:21-28) and the ``BQP1`` varint disk format (programs.py:253-321).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from math import comb
from typing import Iterable, Sequence

from .errors import FormatError, InputError, NoCoveringCircuit, ResourceError

INPUT, CONST0, CONST1 = "input", "const0", "const1"
AND, OR, XOR, ANDNOT, NOT = "and", "or", "xor", "andnot", "not"
SOP_TERM_CAP = 200_000  # core.py:33

OP_ZERO, OP_ONE, OP_AND, OP_OR, OP_XOR, OP_ANDNOT, OP_NOT, OP_RECLAIM = range(8)
_OP_OF = {AND: OP_AND, OR: OP_OR, XOR: OP_XOR, ANDNOT: OP_ANDNOT, NOT: OP_NOT}
_N_OPERANDS = {OP_ZERO: 1, OP_ONE: 1, OP_AND: 3, OP_OR: 3, OP_XOR: 3, OP_ANDNOT: 3, OP_NOT: 2, OP_RECLAIM: 1}


@dataclass
class Circuit:
    """Gate DAG: ``nodes[i] = (kind, a, b)`` in topological order, ordered inputs,
    one output (the reference's Circuit, core.py:38-85)."""

    nodes: list
    inputs: list
    output: int

    @property
    def arity(self) -> int:
        return len(self.inputs)

    def gate_count(self) -> int:
        """Two-input gates reachable from the output (NOT is free, as in the paper)."""
        return sum(1 for i in _reachable(self.nodes, self.output) if self.nodes[i][0] in (AND, OR, XOR, ANDNOT))

    def evaluate(self, bits: Sequence[int]) -> int:
        if len(bits) != len(self.inputs):
            raise InputError("wrong number of input bits")
        val = [0] * len(self.nodes)
        for node, bit in zip(self.inputs, bits):
            val[node] = 1 if bit else 0
        for i, (k, a, b) in enumerate(self.nodes):
            if k == CONST1:
                val[i] = 1
            elif k == AND:
                val[i] = val[a] & val[b]
            elif k == OR:
                val[i] = val[a] | val[b]
            elif k == XOR:
                val[i] = val[a] ^ val[b]
            elif k == ANDNOT:
                val[i] = val[a] & (1 - val[b])
            elif k == NOT:
                val[i] = 1 - val[a]
        return val[self.output]


def _reachable(nodes, root) -> set:
    seen, stack = set(), [root]
    while stack:
        i = stack.pop()
        if i in seen:
            continue
        seen.add(i)
        k, a, b = nodes[i]
        if k in (AND, OR, XOR, ANDNOT):
            stack += [a, b]
        elif k == NOT:
            stack.append(a)
    return seen


class _Builder:
    """Gate builder that folds constants, simplifies x op x, and shares identical
    gates (structural hashing), so the circuits it emits are already optimized."""

    def __init__(self, n: int):
        self.nodes = [(INPUT, -1, -1) for _ in range(n)]
        self.inputs = list(range(n))
        self._memo = {}
        self.zero = self._add((CONST0, -1, -1))
        self.one = self._add((CONST1, -1, -1))

    def _add(self, node) -> int:
        hit = self._memo.get(node)
        if hit is None:
            hit = self._memo[node] = len(self.nodes)
            self.nodes.append(node)
        return hit

    def not_(self, a: int) -> int:
        if a == self.zero:
            return self.one
        if a == self.one:
            return self.zero
        k, x, _ = self.nodes[a]
        return x if k == NOT else self._add((NOT, a, -1))

    def and_(self, a: int, b: int) -> int:
        if self.zero in (a, b):
            return self.zero
        if a == self.one or a == b:
            return b
        if b == self.one:
            return a
        return self._add((AND, min(a, b), max(a, b)))

    def or_(self, a: int, b: int) -> int:
        if self.one in (a, b):
            return self.one
        if a == self.zero or a == b:
            return b
        if b == self.zero:
            return a
        return self._add((OR, min(a, b), max(a, b)))

    def xor(self, a: int, b: int) -> int:
        if a == b:
            return self.zero
        if a == self.zero:
            return b
        if b == self.zero:
            return a
        if a == self.one:
            return self.not_(b)
        if b == self.one:
            return self.not_(a)
        return self._add((XOR, min(a, b), max(a, b)))

    def full_add(self, x: int, y: int, z: int):
        """(sum, carry) of three bits: 2 XOR + carry as (x & y) | (z & (x ^ y))."""
        p = self.xor(x, y)
        return self.xor(p, z), self.or_(self.and_(x, y), self.and_(z, p))

    def geq_const(self, weight: Sequence[int], t: int) -> int:
        """[weight >= t] for an LSB-first binary weight: scan from the LSB, at bit i
        ge = w_i AND ge if t_i = 1 else w_i OR ge (ge starts true: x >= 0)."""
        if t >= 1 << len(weight):
            return self.zero
        ge = self.one
        for i, w in enumerate(weight):
            ge = self.and_(w, ge) if (t >> i) & 1 else self.or_(w, ge)
        return ge

    def finish(self, out: int) -> Circuit:
        return Circuit(list(self.nodes), list(self.inputs), out)


def _check(n: int, t: int):
    if n < 1:
        raise InputError("need at least one input")
    if not 1 <= t <= n:
        raise InputError(f"threshold {t} outside [1, {n}]")


def _weight_bits(n: int) -> int:
    return (2 * n).bit_length() - 1  # m = floor(log2 2N), core.py:240-242


def _sideways_weight(b: _Builder, bits: list) -> list:
    """Carry-save (sideways) sum: columns of equal weight reduced by full adders,
    then half adders, until every column holds one bit."""
    cols = [list(bits)]
    w = 0
    while w < len(cols):
        col = cols[w]
        while len(col) > 1:
            if len(cols) == w + 1:
                cols.append([])
            if len(col) >= 3:
                s, c = b.full_add(col.pop(0), col.pop(0), col.pop(0))
            else:
                x, y = col.pop(0), col.pop(0)
                s, c = b.xor(x, y), b.and_(x, y)
            col.append(s)
            cols[w + 1].append(c)
        w += 1
    return [c[0] if c else b.zero for c in cols]


def _tree_weight(b: _Builder, bits: list) -> list:
    """Balanced tree of ripple-carry adders over binary numbers (leaves: one bit)."""
    nums = [[x] for x in bits]
    while len(nums) > 1:
        nxt = []
        for k in range(0, len(nums) - 1, 2):
            x, y = nums[k], nums[k + 1]
            width = max(len(x), len(y))
            x = x + [b.zero] * (width - len(x))
            y = y + [b.zero] * (width - len(y))
            carry, out = b.zero, []
            for xi, yi in zip(x, y):
                s, carry = b.full_add(xi, yi, carry)
                out.append(s)
            nxt.append(out + [carry])
        if len(nums) % 2:
            nxt.append(nums[-1])
        nums = nxt
    return nums[0]


def build_sideways_sum(n: int, t: int) -> Circuit:
    _check(n, t)
    b = _Builder(n)
    return b.finish(b.geq_const(_sideways_weight(b, b.inputs), t))


def build_tree_adder(n: int, t: int) -> Circuit:
    _check(n, t)
    b = _Builder(n)
    return b.finish(b.geq_const(_tree_weight(b, b.inputs), t))


def build_sorter(n: int, t: int) -> Circuit:
    """Batcher odd-even merge sort (descending; zero pads to a power of two fold
    away); the output is the T-th largest wire."""
    _check(n, t)
    b = _Builder(n)
    size = 1
    while size < n:
        size *= 2
    wires = list(b.inputs) + [b.zero] * (size - n)

    def cmp(i, j):  # larger value (OR) to i, smaller (AND) to j
        wires[i], wires[j] = b.or_(wires[i], wires[j]), b.and_(wires[i], wires[j])

    p = 1
    while p < size:  # the iterative form of Batcher's network
        k = p
        while k >= 1:
            for j in range(k % p, size - k, 2 * k):
                for i in range(min(k, size - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        cmp(i + j, i + j + k)
            k //= 2
        p *= 2
    return b.finish(wires[t - 1])


def build_sop(n: int, t: int, term_cap: int = SOP_TERM_CAP) -> Circuit:
    """OR over all T-subsets of the AND of their members."""
    _check(n, t)
    if comb(n, t) > term_cap:
        raise ResourceError(f"choose({n},{t}) exceeds the term cap {term_cap}")
    from itertools import combinations

    b = _Builder(n)
    out = b.zero
    for subset in combinations(b.inputs, t):
        term = b.one
        for x in subset:
            term = b.and_(term, x)
        out = b.or_(out, term)
    return b.finish(out)


def optimize(circuit: Circuit) -> Circuit:
    """Reachability prune (the builders already fold constants and share gates):
    keep the inputs and the output's fan-in, renumbered in order."""
    keep = _reachable(circuit.nodes, circuit.output) | set(circuit.inputs)
    order = sorted(keep)
    new = {old: i for i, old in enumerate(order)}
    nodes = []
    for old in order:
        k, a, b = circuit.nodes[old]
        nodes.append((k, new.get(a, -1) if a >= 0 else -1, new.get(b, -1) if b >= 0 else -1))
    return Circuit(nodes, [new[i] for i in circuit.inputs], new[circuit.output])


@dataclass
class BitProgram:
    """Straight-line code over slots, ``(opcode, dst, a, b)``, -1 unused
    (programs.py:56-72); inputs occupy slots 0..arity-1."""

    arity: int
    n_slots: int
    result_slot: int
    instructions: list
    peak_slots: int

    @property
    def op_count(self) -> int:
        return sum(1 for ins in self.instructions if ins[0] != OP_RECLAIM)


def compile_circuit(circuit: Circuit) -> BitProgram:
    """Slot allocation in node order with a free list: a value's slot is reclaimed
    right after its last reader (inputs included), so the peak stays near the
    circuit's live width."""
    nodes, out = circuit.nodes, circuit.output
    need = sorted(_reachable(nodes, out))
    uses = {i: 0 for i in need}
    for i in need:
        k, a, b = nodes[i]
        if k in (AND, OR, XOR, ANDNOT):
            uses[a] += 1
            uses[b] += 1
        elif k == NOT:
            uses[a] += 1
    slot = {node: pos for pos, node in enumerate(circuit.inputs)}
    free, ins = [], []
    state = {"next": circuit.arity, "live": circuit.arity, "peak": circuit.arity}

    def alloc():
        if free:
            s = free.pop()
        else:
            s = state["next"]
            state["next"] += 1
        state["live"] += 1
        state["peak"] = max(state["peak"], state["live"])
        return s

    def drop(node):
        s = slot.pop(node)
        free.append(s)
        state["live"] -= 1
        ins.append((OP_RECLAIM, s, -1, -1))

    for node in circuit.inputs:
        if not uses.get(node) and node != out:
            drop(node)
    for i in need:
        k, a, b = nodes[i]
        if k == INPUT:
            continue
        if k in (CONST0, CONST1):
            s = alloc()
            slot[i] = s
            ins.append((OP_ONE if k == CONST1 else OP_ZERO, s, -1, -1))
            continue
        sa = slot[a]
        sb = slot[b] if k != NOT else -1
        s = alloc()
        slot[i] = s
        ins.append((_OP_OF[k], s, sa, sb))
        for operand in ((a,) if k == NOT else (a, b)):
            uses[operand] -= 1
            if uses[operand] == 0 and operand != out and operand in slot:
                drop(operand)
    return BitProgram(circuit.arity, state["next"], slot[out], ins, state["peak"])


_MAGIC = b"BQP1"


def _varint(out: bytearray, v: int):
    while True:
        byte, v = v & 0x7F, v >> 7
        out.append(byte | (0x80 if v else 0))
        if not v:
            return


def dumps_program(p: BitProgram) -> bytes:
    """The reference's on-disk program format (programs.py:253-286)."""
    out = bytearray(_MAGIC)
    for v in (p.arity, p.n_slots, p.result_slot, p.peak_slots, len(p.instructions)):
        _varint(out, v)
    for op, dst, a, b in p.instructions:
        out.append(op)
        for k, v in enumerate((dst, a, b)[: _N_OPERANDS[op]]):
            _varint(out, v)
    return bytes(out)


def loads_program(data: bytes) -> BitProgram:
    if data[:4] != _MAGIC:
        raise FormatError("bad program magic")
    pos = 4

    def rd():
        nonlocal pos
        v = shift = 0
        while True:
            if pos >= len(data):
                raise FormatError("truncated varint")
            byte = data[pos]
            pos += 1
            v |= (byte & 0x7F) << shift
            if not byte & 0x80:
                return v
            shift += 7

    arity, n_slots, result, peak, count = (rd() for _ in range(5))
    ins = []
    for _ in range(count):
        if pos >= len(data):
            raise FormatError("truncated instruction stream")
        op = data[pos]
        pos += 1
        if op not in _N_OPERANDS:
            raise FormatError(f"unknown opcode {op}")
        vals = [rd() for _ in range(_N_OPERANDS[op])] + [-1, -1]
        ins.append((op, vals[0], vals[1], vals[2]))
    return BitProgram(arity, n_slots, result, ins, peak)


BUILDERS = {"sop": build_sop, "sorter": build_sorter, "tree": build_tree_adder, "sideways": build_sideways_sum}


@dataclass(frozen=True)
class PaddingPlan:
    """Answer an (n_req, t_req) query with the stored (n, t) circuit: the real
    inputs plus ``one_pads`` all-ones and ``zero_pads`` all-zero bitmaps
    (library.py:29-46)."""

    n: int
    t: int
    zero_pads: int
    one_pads: int

    def pad_inputs(self, inputs: Sequence) -> list:
        r = max(b.bit_length for b in inputs)
        cls = type(inputs[0])
        padded = list(inputs) + [cls.empty(r)] * self.zero_pads
        if self.one_pads:
            padded += [cls.ones(r)] * self.one_pads
        return padded


def covers(key, n_req: int, t_req: int) -> bool:
    n, t = key
    return n_req <= n and t - (n - n_req) <= t_req <= t


def plan_padding(n_req: int, t_req: int, available: Iterable) -> PaddingPlan:
    """The smallest covering entry, by N then |T - T'| (library.py:54-69)."""
    if n_req < 1 or not 1 <= t_req <= n_req:
        raise InputError(f"bad request ({n_req}, {t_req})")
    cands = [((n, abs(t - t_req), t), (n, t)) for n, t in available if covers((n, t), n_req, t_req)]
    if not cands:
        raise NoCoveringCircuit(f"no stored circuit covers ({n_req}, {t_req})")
    n, t = min(cands)[1]
    return PaddingPlan(n, t, zero_pads=n - n_req - (t - t_req), one_pads=t - t_req)


def tabulation_levels(n_max: int) -> list:
    levels, n = [], 2
    while n <= n_max:
        levels.append(n)
        n *= 2
    if n_max >= 2 and n_max not in levels:
        levels.append(n_max)
    return levels


def program_path(cache_dir: str | None, builder: str, n: int, t: int) -> str | None:
    """Cache file name of a tabulated program (library.py:130-133)."""
    if cache_dir is None:
        return None
    return os.path.join(cache_dir, f"{builder}_n{n}_t{t}.bqp")
