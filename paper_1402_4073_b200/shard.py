"""Word-range sharding of a threshold / symmetric query across GPUs.

The reference is single-threaded but names the scale-out
scheme: horizontal fragmentation by row range, which its
word-batch evaluator realises (circuits/programs.py:196-237).  Output word w
depends only on input words w, so rank g of G owns the word range
``shard_range(total, G, g)`` of every input bitmap and of the result; no input
data crosses GPUs.  The one exchange is the result popcount (an 8-byte
all-reduce per query); assembling the full result on one rank is optional
(``gather_result``).

One process per GPU (torchrun), ``torch.distributed`` with NCCL for the
all-reduce.  ``ShardedQuery`` takes an ``evaluate`` hook so the host-side
logic (partition, reduction, gather) is testable with gloo on CPU.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist

from .bitmaps import word_count
from .errors import InputError

TILE_WORDS = 512  # kernel tile; shard boundaries are tile aligned (and even, for 16-byte loads)
RLE_TILE_WORDS = 1024  # RLE tile (K3 directory granularity): RLE shard boundaries


def shard_range(total_words: int, world: int, rank: int, align: int = TILE_WORDS) -> tuple[int, int]:
    """Contiguous, ``align``-aligned word range [begin, end) owned by ``rank``.

    Ranges of ranks 0..world-1 tile [0, total_words) exactly, with sizes
    differing by at most one alignment unit."""
    if world < 1 or not 0 <= rank < world:
        raise InputError(f"bad rank {rank} of {world}")
    if align < 2 or align % 2:
        raise InputError("alignment must be a positive even number of words")
    units = (total_words + align - 1) // align
    per, extra = divmod(units, world)
    first = rank * per + min(rank, extra)
    count = per + (1 if rank < extra else 0)
    begin = min(total_words, first * align)
    end = min(total_words, (first + count) * align)
    return begin, end


def local_bit_length(r_bits: int, begin: int, end: int) -> int:
    """Bit length of the window [begin, end) words of an r_bits-long result."""
    return max(0, min(r_bits - 64 * begin, 64 * (end - begin)))


def local_words(n_words: int, begin: int, end: int) -> int:
    """Valid words of an input (``n_words`` long globally) inside [begin, end)."""
    return max(0, min(n_words, end) - begin)


class ShardedQuery:
    """This rank's shard of a query over N bitmaps, plus the cross-rank reduction.

    ``local_inputs``: per input, a 1-D int64 device tensor holding its words
    [begin, begin + local_words) (the rank's slice).  With ``rle=True`` they are
    instead the WHOLE compressed streams, replicated on every rank (SURVEY
    §8(e): ~2.3 GiB at C4); each rank decodes only its word range, whose bounds
    are then multiples of the 1024-word RLE tile.  ``r_bits`` is the GLOBAL
    result bit length.  ``evaluate(kind, arg, inputs, r_local) -> (words, popcount)``
    overrides the device evaluation (tests use a CPU oracle with gloo)."""

    def __init__(self, local_inputs: Sequence, r_bits: int, world: int | None = None, rank: int | None = None,
                 group=None, evaluate: Callable | None = None, align: int = TILE_WORDS, rle: bool = False):
        self.group = group
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if dist.is_initialized() else 0)
        self.r_bits = int(r_bits)
        self.total_words = word_count(self.r_bits)
        self.rle = bool(rle)
        if self.rle:
            align = max(align, RLE_TILE_WORDS)
            if align % RLE_TILE_WORDS:
                raise InputError(f"RLE shard alignment must be a multiple of {RLE_TILE_WORDS} words")
        self.align = align
        self.begin, self.end = shard_range(self.total_words, self.world, self.rank, align)
        self.r_local = local_bit_length(self.r_bits, self.begin, self.end)
        self.inputs = list(local_inputs)
        self._evaluate = evaluate
        self._q = None
        if evaluate is None:
            if self.rle:
                from .engine import RleQuery
                self._q = RleQuery(self.inputs, self.r_bits, word_range=(self.begin, self.end))
            else:
                from .engine import ThresholdQuery
                self._q = ThresholdQuery(self.inputs, self.r_local)

    @property
    def n(self) -> int:
        return len(self.inputs)

    def _local(self, kind, arg, out=None, popcnt=None, stream=None):
        if self._evaluate is not None:
            return self._evaluate(kind, arg, self.inputs, self.r_local)
        if kind == "threshold":
            return self._q.threshold(arg, out, popcnt, stream=stream)
        return self._q.symmetric(arg, out, popcnt, stream=stream)

    def threshold(self, t: int, out=None, popcnt=None, stream=None, reduce: bool = True):
        """Evaluate this rank's words; all-reduce the popcount when ``reduce``."""
        if not 1 <= t <= self.n:
            raise InputError(f"threshold {t} outside [1, {self.n}]")
        words, pc = self._local("threshold", t, out, popcnt, stream)
        if reduce:
            pc = allreduce_popcount(pc, self.group)
        return words, pc

    def symmetric(self, accept, out=None, popcnt=None, stream=None, reduce: bool = True):
        words, pc = self._local("symmetric", accept, out, popcnt, stream)
        if reduce:
            pc = allreduce_popcount(pc, self.group)
        return words, pc

    def gather_result(self, local_out: torch.Tensor, dst: int | None = 0):
        """Assemble the full result (``dst`` rank, or every rank when dst is None)."""
        return gather_result(local_out[: self.end - self.begin], self.total_words, self.world, self.rank,
                             self.group, dst, self.align)


def allreduce_popcount(pc: torch.Tensor, group=None) -> torch.Tensor:
    """Sum per-rank popcounts (int64 tensor) over the group; no-op on one rank."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(pc, op=dist.ReduceOp.SUM, group=group)
    return pc


def gather_result(local: torch.Tensor, total_words: int, world: int, rank: int, group=None, dst=0,
                  align: int = TILE_WORDS):
    """Concatenate every rank's result words in rank order.

    Shards differ in length by at most one tile, so each is padded to the
    largest before all_gather and the padding is dropped after."""
    if world == 1 or not dist.is_initialized():
        return local
    sizes = [e - b for b, e in (shard_range(total_words, world, g, align) for g in range(world))]
    width = max(sizes)
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if dst is not None and rank != dst:
        return None
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])
