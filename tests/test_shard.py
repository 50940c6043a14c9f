"""Multi-GPU host logic on CPU: word-range shard plans, and the cross-rank
popcount all-reduce + result gather at world size 2 over gloo.  The per-rank
evaluation is injected (CPU oracle) because this container has no GPU; the
device evaluation of a shard is covered by tests/test_gpu_threshold.py
(test_word_range_shards_tile_the_result)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_4073_b200.shard import ShardedQuery, local_bit_length, local_words, shard_range


@pytest.mark.parametrize("total", [0, 1, 2, 511, 512, 513, 4096, 100003, 1 << 22])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_tile_exactly(total, world):
    prev = 0
    sizes = []
    for g in range(world):
        b, e = shard_range(total, world, g)
        assert b == prev and e >= b
        assert b % 512 == 0 or b == total
        sizes.append(e - b)
        prev = e
    assert prev == total
    full = [s for s in sizes if s]
    if len(full) > 1:
        assert max(full[:-1]) - min(full[:-1]) <= 512


def test_local_geometry():
    r = 64 * 1000 - 5
    assert local_bit_length(r, 0, 512) == 64 * 512
    assert local_bit_length(r, 512, 1000) == r - 64 * 512
    assert local_words(700, 512, 1000) == 188
    assert local_words(100, 512, 1000) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    rng = np.random.default_rng(5)
    n, r = 11, 64 * 3000 - 17
    nw = (r + 63) // 64
    full = []
    for i in range(n):
        a = rng.integers(0, 2**64, size=nw, dtype=np.uint64) & rng.integers(0, 2**64, size=nw, dtype=np.uint64)
        a[-1] &= np.uint64((1 << (r % 64)) - 1)
        full.append(a[: nw - 97 * i])  # ragged
    b, e = shard_range(nw, world, rank)
    local = [torch.from_numpy(a[b:min(e, a.size)].view(np.int64).copy()) for a in full]

    def evaluate(kind, arg, inputs, r_local):
        arrs = [t.numpy().view(np.uint64) for t in inputs]
        if kind == "threshold":
            words = O.scan_count(arrs, r_local, arg)
        else:
            words = O.scan_count_symmetric(arrs, r_local, arg)
        pc = int(np.unpackbits(words.view(np.uint8)).sum())
        return torch.from_numpy(words.view(np.int64).copy()), torch.tensor([pc], dtype=torch.int64)

    q = ShardedQuery(local, r, evaluate=evaluate)
    assert (q.begin, q.end) == (b, e)
    ok = True
    for t in (1, 3, 6, 11):
        words, pc = q.threshold(t)
        whole = q.gather_result(words, dst=0)
        if rank == 0:
            exp = O.scan_count(full, r, t)
            ok &= np.array_equal(whole.numpy().view(np.uint64), exp)
            ok &= int(pc.item()) == int(np.unpackbits(exp.view(np.uint8)).sum())
    acc = [2 <= k <= 5 for k in range(n + 1)]
    words, pc = q.symmetric(acc)
    whole = q.gather_result(words, dst=None)
    exp = O.scan_count_symmetric(full, r, acc)
    ok &= np.array_equal(whole.numpy().view(np.uint64), exp)
    ok &= int(pc.item()) == int(np.unpackbits(exp.view(np.uint8)).sum())
    with open(f"{result_path}.{rank}", "w") as fp:
        fp.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo(tmp_path):
    world = 2
    path = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    for g in range(world):
        assert open(f"{path}.{g}").read() == "ok"


def _rle_worker(rank, world, port, result_path):
    """RLE shards: every rank holds the whole compressed streams and evaluates only
    its 1024-aligned word window."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    rng = np.random.default_rng(9)
    n, r = 7, 64 * 5000 - 3
    nw = (r + 63) // 64
    streams = []
    for i in range(n):
        w = rng.integers(0, 2**64, size=nw, dtype=np.uint64) & rng.integers(0, 2**64, size=nw, dtype=np.uint64)
        w[rng.integers(0, nw, size=nw // 2)] = 0  # runs of zeros
        w[-1] &= np.uint64((1 << (r % 64)) - 1)
        streams.append(O.rle_compress(O.trim(w), r))

    def evaluate(kind, arg, inputs, r_local):
        # the device query decodes only [begin, end) of the whole streams: the oracle
        # decodes everything and keeps that window
        words = O.cdom_threshold(inputs, r, arg)[q.begin:q.end]
        pc = int(np.unpackbits(words.view(np.uint8)).sum())
        return torch.from_numpy(words.view(np.int64).copy()), torch.tensor([pc], dtype=torch.int64)

    q = ShardedQuery(streams, r, evaluate=evaluate, rle=True)
    b, e = shard_range(nw, world, rank, 1024)
    ok = (q.begin, q.end) == (b, e) and b % 1024 == 0 and q.r_local == local_bit_length(r, b, e)
    for t in (1, 2, 4, 7):
        words, pc = q.threshold(t)
        whole = q.gather_result(words, dst=None)
        exp = O.cdom_threshold(streams, r, t)
        ok &= np.array_equal(whole.numpy().view(np.uint64), exp)
        ok &= int(pc.item()) == int(np.unpackbits(exp.view(np.uint8)).sum())
    with open(f"{result_path}.{rank}", "w") as fp:
        fp.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo_rle(tmp_path):
    world = 2
    path = str(tmp_path / "res")
    mp.spawn(_rle_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    for g in range(world):
        assert open(f"{path}.{g}").read() == "ok"
