"""Benchmark: input GB/s of T-of-N threshold queries on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1], "C2"): N=64 uncompressed bitmaps
of r=2^28 bits per GPU (2 GiB of input per GPU), per-bitmap densities drawn
from U[0.01, 0.5], T swept over {1, 2, 16, 32, 64}.  One step = the five
queries over the resident inputs (5 x 2 GiB of input bytes per GPU) plus the
8-byte-per-query popcount all-reduce across ranks.  Inputs (2 GiB) are far
larger than L2 (126 MB), so no flush is needed between steps.

Multi-GPU: one process per GPU (torchrun); rank g owns words
[g*2^22, (g+1)*2^22) of global bitmaps of world*2^28 bits (weak scaling, no
data-path collective; only the popcount all-reduce).

Lines printed by rank 0 (one JSON object):
  value       device-resident throughput (input bytes / max-over-ranks time)
  e2e         the same metric through the public host-buffer API
              (paper_1402_4073_b200.sweep_host, pinned host inputs, H2D + D2H
              inside the timed region)
  roofline    the counting kernel's achieved HBM GB/s (algorithmic bytes per
              launch / mean CUDA-event launch time) vs MEASURED_PEAKS.json
  cpu_baseline the CPU oracle port timed on this host's cores (rank 0, N=1)

``--impl reference`` times the reference algorithm's CPU port (oracle/, the
reference is Python and has no native build) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "input GB/s (and fraction of HBM peak) for T-of-N threshold queries at 1/2/4/8 B200"
SEED = 1402
C2_N = 64
C2_WORDS = 1 << 22          # words per bitmap per GPU (r = 2^28 bits)
C2_TS = (1, 2, 16, 32, 64)
DENS_LO, DENS_HI = 655, 32768   # round(0.01 * 2^16), 0.5 * 2^16


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fp:
            d = json.load(fp)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """Per-launch DRAM bytes of the counting kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fp:
            d = json.load(fp)
        return d.get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.gpu), "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path or not os.path.exists(self.path):
            return None
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fp:
            for line in fp:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for name, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def physical_gpu_index(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        items = [v.strip() for v in vis.split(",") if v.strip()]
        if local < len(items) and items[local].isdigit():
            return int(items[local])
    return local


# ---------------------------------------------------------------------------
# CPU side (oracle port): used for cpu_baseline and --impl reference

def cpu_windows(nwin: int, win_words: int, world_rank_offset: int = 0):
    """Host copies of ``nwin`` distinct C2 windows (N x win_words each) of the same
    seeded inputs as the GPU arm (bitmap i, global words), generated by the oracle's
    independent restatement of the generator (oracle/bq_oracle.c orc_gen_*), so the
    CPU legs never load libbq.so."""
    from oracle import oracle as O

    qs = [O.gen_density_q16(SEED, i, DENS_LO, DENS_HI) for i in range(C2_N)]
    wins = []
    stride = C2_WORDS // nwin
    for k in range(nwin):
        w0 = world_rank_offset + k * stride
        wins.append([O.gen_bernoulli(SEED, i, qs[i], w0, win_words) for i in range(C2_N)])
    return wins


def _oracle_build() -> str:
    from oracle import oracle as O

    return ("AVX-512 build (x86-64-v4)" if O.library_path().endswith("_avx512.so")
            else "AVX2 build (x86-64-v3)")


def cpu_port_run(wins, steps: int, warmup: int, threads: int):
    """Time the oracle's CPU port of the reference algorithms (wide_or / wide_and /
    csv_threshold, oracle/bq_oracle.c) over the windows, 5 queries per step."""
    from oracle import oracle as O

    win_words = wins[0][0].size
    r = 64 * win_words
    for s in range(warmup):
        for t in C2_TS:
            O.threshold_port(wins[s % len(wins)], r, t, threads)
    t0 = time.perf_counter()
    for s in range(steps):
        for t in C2_TS:
            O.threshold_port(wins[s % len(wins)], r, t, threads)
    dt = time.perf_counter() - t0
    nbytes = steps * len(C2_TS) * C2_N * win_words * 8
    return nbytes / dt / 1e9, dt


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(budget_s: float = 12.0):
    threads = host_threads()
    win_words = 1 << 16
    wins = cpu_windows(8, win_words)
    # calibrate: one step, then size the step count to the time budget
    gbs, dt = cpu_port_run(wins, 1, 1, threads)
    steps = max(2, int(budget_s / max(dt, 1e-3)))
    gbs, dt = cpu_port_run(wins, steps, 0, threads)
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"C2 windows: 8 x (N=64 x 2^16 words), T in {list(C2_TS)}, {steps} steps "
                      f"({dt:.1f} s) of oracle/bq_oracle.c orc_threshold_port (wide_or / wide_and / "
                      f"csv_threshold, OpenMP {threads} threads, {_oracle_build()})"}


# ---------------------------------------------------------------------------
# the stock reference Python (oracle/_ref, installed by build()): context numbers

REF_ALGOS = ("scancount", "looped", "csvckt", "ssum", "treeadd")


def _ref_window_worker(job):
    """One process: the reference's own algorithms (its registry, single-threaded as
    shipped) over one C2 window, every T of the sweep; returns {algo: seconds}."""
    w0, win_words, algos = job
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    from bitquorum import bitmaps as rbm
    from bitquorum.bench import competitions as comp

    from oracle import oracle as O

    qs = [O.gen_density_q16(SEED, i, DENS_LO, DENS_HI) for i in range(C2_N)]
    ins = [rbm.UncompressedBitmap([int(w) for w in O.gen_bernoulli(SEED, i, qs[i], w0, win_words)], 64 * win_words)
           for i in range(C2_N)]
    ctx = comp.RunContext()
    out = {}
    for name in algos:
        algo = comp.ALGORITHMS[name]
        dt = 0.0
        for t in C2_TS:
            if name == "csvckt" and not 2 <= t < C2_N:
                algo_t = comp.ALGORITHMS["looped"]  # csv's contract is 2 <= T < N (bitparallel.py:63-64)
            else:
                algo_t = algo
            if name in ("ssum", "treeadd"):  # circuits are built untimed, as the reference's RunContext does
                ctx.program("sideways" if name == "ssum" else "tree", C2_N, t)
            t0 = time.perf_counter()
            algo_t.run(ins, t, ctx)
            dt += time.perf_counter() - t0
        out[name] = dt
    return out


def reference_python_baseline():
    """SURVEY §8(d) / BASELINE.md §3 items 1-2: the reference package as shipped,
    on this host.  Each algorithm over one 2^12-word C2 window (64 bitmaps, 2 MiB)
    for the whole T sweep on one core, and the best per-T algorithm on K =
    host-thread processes over disjoint windows (exact: the query is word-local).
    Returns None when the reference is not installed (oracle/install_ref.sh)."""
    if not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "bitquorum")):
        return None
    import multiprocessing as mp

    win = 1 << 12
    nbytes = len(C2_TS) * C2_N * win * 8
    one = _ref_window_worker((0, win, REF_ALGOS))
    per_algo = {k: round(nbytes / v / 1e9, 5) for k, v in one.items()}
    best = min(one, key=one.get)
    k = host_threads()
    with mp.get_context("spawn").Pool(k) as pool:
        res = pool.map(_ref_window_worker, [((j + 1) * (C2_WORDS // (k + 1)), win, (best,)) for j in range(k)])
    slowest = max(r[best] for r in res)
    return {"unit": "GB/s", "one_core": per_algo, "best_algorithm": best,
            "one_core_best": per_algo[best],
            "k_processes": {"processes": k, "value": round(k * nbytes / slowest / 1e9, 5),
                            "note": "K windows over the slowest process's in-process query time (inputs "
                                    "built and circuits compiled untimed in every process)"},
            "sample": f"C2 windows of 2^12 words x 64 bitmaps (2 MiB), T in {list(C2_TS)}; csvckt falls back to "
                      "looped where its 2 <= T < N contract excludes T; circuits built untimed",
            "source": "reference bitquorum as shipped (oracle/_ref), its ALGORITHMS registry"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(max(1, args.gpus))))
    if rank != 0:
        return 0
    threads = host_threads()
    win_words = 1 << 16
    wins = cpu_windows(16, win_words)
    gbs, dt = cpu_port_run(wins, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1000 / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (bq_gen Bernoulli, seed 1402)",
        "config": {"workload": "C2 sample: N=64 bitmaps, 16 distinct windows of 2^16 words (512 MiB), "
                               "T sweep {1,2,16,32,64}; one step = 5 queries over one window",
                   "n_bitmaps": C2_N, "ts": list(C2_TS),
                   "same_config_as_gpu_arm": False,
                   "sample_note": "bounded sample of the GPU arm's C2 workload (same seeded bitmaps, same metric and "
                                  "T sweep): word windows instead of the full 2 GiB, since cost is linear in words "
                                  "(PAPER.md:283-298); the windows (512 MiB) exceed the host caches"},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": "reference algorithms (wide_or / wide_and / csv_threshold) restated in C "
                                   f"(oracle/bq_oracle.c, {_oracle_build()}), OpenMP over word batches, on C2 windows"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_reference_python:
        line["reference_python"] = reference_python_baseline()
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU side

def _dist_setup(torch, dist):
    """One process per GPU: (rank, world, device index).  The collective backend is
    NCCL.  Functional checks of the multi-rank flow on a one-GPU box may set
    BQ_BENCH_BACKEND=gloo and BQ_BENCH_SHARE_GPU=1 (ranks then share device
    LOCAL_RANK mod device_count; their numbers are not measurements)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BQ_BENCH_SHARE_GPU") == "1":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BQ_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1402_4073_b200 as bq
    from paper_1402_4073_b200 import _lib

    rank, world, local = _dist_setup(torch, dist)
    lib = _lib.load()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    n, nw = C2_N, C2_WORDS
    pitch = nw + args.pad_words
    w0 = rank * nw
    r_local = 64 * nw
    qs = [lib.bq_gen_density_q16(SEED, i, DENS_LO, DENS_HI) for i in range(n)]
    data = torch.empty((n, pitch), dtype=torch.int64, device=dev)
    qarr = np.asarray(qs, dtype=np.uint32)
    _lib.check(lib.bq_gen_bernoulli_rows(SEED, 0, n, qarr.ctypes.data, w0, nw, data.data_ptr(), pitch, sh))
    rows = [data[i, :nw] for i in range(n)]
    query = bq.ThresholdQuery(rows, r_local)
    outs = torch.empty((len(C2_TS), nw), dtype=torch.int64, device=dev)
    pcs = torch.zeros(len(C2_TS), dtype=torch.int64, device=dev)

    def step(ev=None):
        pcs.zero_()
        for k, t in enumerate(C2_TS):
            if ev is not None:
                ev[k][0].record(stream)
            query.threshold(t, outs[k], pcs[k:k + 1], stream=stream)
            if ev is not None:
                ev[k][1].record(stream)
        if world > 1:
            dist.all_reduce(pcs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    kev = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
            for _ in C2_TS] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(physical_gpu_index(local)) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        for s in range(args.steps):
            step()  # no instrumentation inside the timed region: per-launch events cost ~3 us each
        stop.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    # the average launch over the timed region (the per-step popcount reset included)
    launch_ms = [elapsed_ms / (args.steps * len(C2_TS))]
    # per-threshold breakdown: a diagnostic pass after the timed region, each launch between events
    diag = min(args.steps, 20)
    for s in range(diag):
        step(kev[s])
    torch.cuda.synchronize()
    per_t_ms = {t: statistics.mean(kev[s][k][0].elapsed_time(kev[s][k][1]) for s in range(diag))
                for k, t in enumerate(C2_TS)}
    mt = torch.tensor([elapsed_ms, statistics.mean(launch_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
    elapsed_ms, mean_launch_ms = float(mt[0]), float(mt[1])
    final_pc = pcs.tolist()

    in_bytes_step = world * len(C2_TS) * n * nw * 8
    value = in_bytes_step * args.steps / (elapsed_ms / 1e3) / 1e9
    algo_bytes_launch = n * nw * 8 + nw * 8
    achieved = algo_bytes_launch / (mean_launch_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()

    # --- end to end through the public host-buffer API -------------------------
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty((n, nw), dtype=torch.int64, pin_memory=True)
        host_in.copy_(data[:, :nw])
        h_in = [host_in[i].numpy().view(np.uint64) for i in range(n)]
        host_out = torch.empty((len(C2_TS), nw), dtype=torch.int64, pin_memory=True)
        h_out = [host_out[k].numpy().view(np.uint64) for k in range(len(C2_TS))]
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        chunk_words = (args.e2e_chunk_mib << 20) // (8 * n) if args.e2e_chunk_mib else 0
        for _ in range(max(1, min(args.warmup, 2))):
            bq.sweep_host(h_in, r_local, list(C2_TS), outs=h_out, device=local, chunk_words=chunk_words)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            _, pops = bq.sweep_host(h_in, r_local, list(C2_TS), outs=h_out, device=local, chunk_words=chunk_words)
            if world > 1:
                pt = torch.tensor(pops, dtype=torch.int64, device=dev)
                dist.all_reduce(pt)
        e2e_s = time.perf_counter() - t0
        et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_s = float(et[0])
        # parity of the host path with the device path on this step's result
        ok = all(np.array_equal(h_out[k], outs[k].cpu().numpy().view(np.uint64)) for k in range(len(C2_TS)))
        e2e = {"value": round(in_bytes_step * e2e_steps / e2e_s / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": n * nw * 8, "d2h_bytes_per_step": len(C2_TS) * nw * 8 + len(C2_TS) * 8,
               "steps": e2e_steps, "ms_per_step": round(e2e_s * 1e3 / e2e_steps, 3),
               "api": "paper_1402_4073_b200.sweep_host -> bq_sweep_host (pinned host in/out)",
               "matches_device_result": bool(ok)}

    # --- C5 strong scaling (BASELINE configs[4]): the sharded majority query --------
    c5 = None
    if not args.no_c5:
        import types

        ctx = types.SimpleNamespace(world=world, rank=rank, dist=dist, cpu=False)
        l5 = run_c5(args, torch, bq, lib, dev, stream, ctx)
        red = torch.tensor([l5["_rank_ms"], float(l5["_rank_bytes"]), float(l5["popcount"])], dtype=torch.float64,
                           device=dev)
        mx = red.clone()
        if world > 1:
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(red, op=dist.ReduceOp.SUM)
        job_ms, job_bytes = float(mx[0]), float(red[1])
        c5 = {"value": round(job_bytes / (job_ms / 1e3) / 1e9, 3), "unit": "GB/s", "scaling": "strong",
              "query_ms": round(job_ms, 4), "n_gpus": world, "input_bytes": int(job_bytes),
              "waves_per_rank": l5["config"]["waves_per_rank"], "popcount": int(red[2]),
              "roofline_frac": l5["roofline"]["frac"],
              "workload": "C5: N=511, r=2^32 bits, p=0.5, T=256 (256 GiB) split by word range over the ranks; "
                          "each rank runs its shard as waves of <= 32 GiB (8 waves at N=1, 1 at N=8); query_ms = "
                          "max over ranks of the summed per-wave query times, each query followed by the popcount "
                          "all-reduce (inside the timed launches)"}
        del l5
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(elapsed_ms / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic: counter-based Bernoulli generator (csrc/bq_gen.h), seed 1402, "
                    "per-bitmap density U[0.01,0.5] quantized to q/2^16",
            "config": {"workload": "C2 (BASELINE configs[1]): N=64 bitmaps x r=2^28 bits per GPU (2 GiB input/GPU), "
                                   "T sweep {1,2,16,32,64}; step = 5 queries + popcount all-reduce",
                       "n_bitmaps": n, "r_bits_per_gpu": 64 * nw, "ts": list(C2_TS),
                       "global_r_bits": 64 * nw * world, "row_pitch_words": pitch,
                       "l2": "inputs 2 GiB/GPU > 126 MB L2; no flush needed",
                       "parallelism": f"word-range shards x{world} GPUs, popcount all-reduce only"},
            "per_query_ms": {str(t): round(v, 5) for t, v in per_t_ms.items()},
            "per_query_ms_note": "diagnostic pass after the timed region, each launch between CUDA events; "
                                 "roofline.mean_launch_ms = timed region / launches (popcount resets included)",
            "popcounts": {str(t): int(p) for t, p in zip(C2_TS, final_pc)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic("c2"),
                         "kernel": "bq::count_kernel (all 5 T; OR/AND/comparator epilogues)",
                         "algorithmic_bytes_per_launch": algo_bytes_launch,
                         "mean_launch_ms": round(mean_launch_ms, 5), "peak_source": peak_src},
            "gpu_launches": len(C2_TS) * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "c5_strong_scaling": c5,
        }
        cl = clocks.summary()
        line["clocks"] = cl
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# the other BASELINE configs (parity-test cases; extra lines via --workload)

def _l2_flush(scratch):
    """Evict L2 by READING a buffer larger than it (clean lines, no write-backs
    charged to the next kernel)."""
    scratch.view(-1).sum(dtype=scratch.dtype if scratch.dtype.is_floating_point else None)


def _timed_launches(torch, launch, steps, warmup, stream, flush=None):
    """Run `launch()` (which enqueues kernels on `stream`) warmup+steps times;
    return per-launch CUDA-event times in ms.  `flush()` (L2 flush) runs
    between launches outside the events; without a flush the launches run back
    to back between one event pair and each gets the average."""
    for _ in range(warmup):
        if flush:
            flush()
        launch()
    torch.cuda.synchronize()
    if not flush:  # back-to-back launches: one event pair around all of them (no instrumentation inside)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            launch()
        b.record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) / steps] * steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s in range(steps):
        flush()
        ev[s][0].record(stream)
        launch()
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def _line(workload, value, per_launch_ms, algo_bytes, steps, warmup, config, extra=None, unit="GB/s",
          traffic_key=None):
    peak, peak_src = measured_peak()
    mean_ms = statistics.mean(per_launch_ms)
    achieved = algo_bytes / (mean_ms / 1e3) / 1e9
    line = {"metric": METRIC, "workload": workload, "value": round(value, 3), "unit": unit, "n_gpus": 1,
            "steps": steps, "warmup": warmup, "ms_per_step": round(sum(per_launch_ms) / len(per_launch_ms), 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (csrc/bq_gen.h generators, seed 1402)", "config": config,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic(traffic_key or workload),
                         "algorithmic_bytes_per_launch": algo_bytes, "mean_launch_ms": round(mean_ms, 5),
                         "median_launch_ms": round(statistics.median(per_launch_ms), 5),
                         "min_launch_ms": round(min(per_launch_ms), 5),
                         "peak_source": peak_src},
            "gpu_launches": len(per_launch_ms)}
    if extra:
        line.update(extra)
    return line


def run_c1(args, torch, bq, lib, dev, stream, ctx):
    """Config 1: N=8, r=2^20, p=0.1, T=3 (1 MiB: L2-resident, launch-bound)."""
    n, nw, t = 8, 1 << 14, 3
    data = torch.empty((n, nw), dtype=torch.int64, device=dev)
    qarr = np.full(n, 6554, dtype=np.uint32)
    _lib_check(lib.bq_gen_bernoulli_rows(SEED, 0, n, qarr.ctypes.data, 0, nw, data.data_ptr(), nw, stream.cuda_stream))
    q = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
    out = torch.empty(nw, dtype=torch.int64, device=dev)
    pc = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    ms = _timed_launches(torch, lambda: q.threshold(t, out, pc, stream=stream), args.steps, args.warmup, stream,
                         flush=lambda: _l2_flush(scratch))
    # the floor of this timing method: a one-element kernel between the same events after the same flush
    one = torch.zeros(1, dtype=torch.int64, device=dev)
    floor_ms = _timed_launches(torch, lambda: one.add_(1), args.steps, args.warmup, stream,
                               flush=lambda: _l2_flush(scratch))
    in_bytes = n * nw * 8
    from oracle import oracle as O
    host = [data[i].cpu().numpy().view(np.uint64) for i in range(n)]
    t0 = time.perf_counter()
    reps = 0
    while ctx.cpu and time.perf_counter() - t0 < 2.0:
        O.threshold_port(host, 64 * nw, t, host_threads())
        reps += 1
    cpu_gbs = reps * in_bytes / (time.perf_counter() - t0) / 1e9
    exact = np.array_equal(out.cpu().numpy().view(np.uint64), O.scan_count(host, 64 * nw, t))
    line = _line("c1", in_bytes / (statistics.mean(ms) / 1e3) / 1e9, ms, in_bytes + nw * 8, args.steps, args.warmup,
                 {"workload": "C1: N=8, r=2^20 bits, p=0.1 (q=6554), T=3; L2 flushed (256 MB read) between launches",
                  "n_bitmaps": n, "r_bits": 64 * nw, "t": t},
                 {"matches_oracle": bool(exact),
                  "timing_floor_ms": round(statistics.median(floor_ms), 5),
                  "timing_floor_note": "median of a one-element kernel timed the same way (events around one "
                                       "launch after a 256 MB L2 flush): C1 is launch/latency bound",
                  "cpu_baseline": {"value": round(cpu_gbs, 3), "unit": "GB/s", "cores": host_threads(), "kind": "port",
                                   "sample": "full C1, orc_threshold_port (csv_threshold port), 2 s"}})
    line["_rank_bytes"] = in_bytes  # replicas at N > 1
    return line


def run_c3(args, torch, bq, lib, dev, stream, ctx):
    """Config 3: N=256, r=2^26, p=0.05, accept = count in [2, 10] (2 GiB)."""
    n, nw = 256, 1 << 20
    pitch = nw + args.pad_words
    data = torch.empty((n, pitch), dtype=torch.int64, device=dev)
    qarr = np.full(n, 3277, dtype=np.uint32)
    _lib_check(lib.bq_gen_bernoulli_rows(SEED, 0, n, qarr.ctypes.data, 0, nw, data.data_ptr(), pitch,
                                         stream.cuda_stream))
    q = bq.ThresholdQuery([data[i, :nw] for i in range(n)], 64 * nw)
    acc = [2 <= k <= 10 for k in range(n + 1)]
    out = torch.empty(nw, dtype=torch.int64, device=dev)
    pc = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = _timed_launches(torch, lambda: q.symmetric(acc, out, pc, stream=stream), args.steps, args.warmup, stream)
    pc.zero_()
    q.symmetric(acc, out, pc, stream=stream)
    in_bytes = n * nw * 8
    from oracle import oracle as O
    win = 1 << 14
    host = [data[i, :win].cpu().numpy().view(np.uint64) for i in range(n)]
    exact = np.array_equal(out[:win].cpu().numpy().view(np.uint64), O.scan_count_symmetric(host, 64 * win, acc))
    t0 = time.perf_counter()
    reps = 0
    while ctx.cpu and time.perf_counter() - t0 < 5.0:
        O.symmetric_port(host, 64 * win, acc, host_threads())
        reps += 1
    cpu_gbs = reps * n * win * 8 / (time.perf_counter() - t0) / 1e9
    line = _line("c3", in_bytes / (statistics.mean(ms) / 1e3) / 1e9, ms, in_bytes + nw * 8, args.steps, args.warmup,
                 {"workload": "C3: N=256, r=2^26 bits, p=0.05 (q=3277), accept = [2 <= count <= 10] (2 GiB)",
                  "n_bitmaps": n, "r_bits": 64 * nw, "accept": "interval [2,10]"},
                 {"matches_oracle_window": bool(exact), "popcount": int(pc.item()),
                  "cpu_baseline": {"value": round(cpu_gbs, 3), "unit": "GB/s", "cores": host_threads(), "kind": "port",
                                   "sample": "C3 window N=256 x 2^14 words, orc_symmetric_port, 5 s"}})
    line["_rank_bytes"] = in_bytes  # replicas at N > 1
    return line


def _markov_streams(lib, n, r, m1, m0, threads):
    """Generate n C4 streams on the host (ctypes releases the GIL -> threads)."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    def one(i):
        cap = max(4096, int(r / 64 * 0.2))
        while True:
            buf = np.empty(cap, dtype=np.uint64)
            nout = ctypes.c_uint64(0)
            rc = lib.bq_gen_markov_rle(SEED, i, r, m1, m0, buf.ctypes.data, cap, ctypes.byref(nout))
            if rc == 0:
                return buf[: nout.value].copy()
            cap = int(nout.value) + 16

    with ThreadPoolExecutor(max(1, threads)) as ex:
        return list(ex.map(one, range(n)))


def _oracle_markov_streams(n, r, m1, m0, threads):
    """The same C4 streams from the oracle's generator restatement (CPU legs only)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    with ThreadPoolExecutor(max(1, threads)) as ex:
        return list(ex.map(lambda i: O.gen_markov_rle(SEED, i, r, m1, m0), range(n)))


def run_c4(args, torch, bq, lib, dev, stream, ctx):
    """Config 4: N=1024 RLE bitmaps, r=2^30, one-runs mean 256 bits, zero-runs mean
    12544 (density 0.02, interpretation A of SURVEY App. B), T=50; output uncompressed.

    value = EWAH input bytes / FRESH-query time: a new query over device-resident
    streams, i.e. the K3 directory pass plus the first evaluation (K4), which reads
    the streams themselves.  A reused query's later evaluations run K4s on the
    tile-sliced layout derived from the streams (built once, at the second
    evaluation); they are reported separately under ``repeated_query`` with the
    bytes K4s actually moves and the layout build cost."""
    n, r, t = 1024, 1 << 30, args.c4_t
    m1, m0 = 256.0, 12544.0
    t_gen = time.perf_counter()
    streams = _markov_streams(lib, n, r, m1, m0, host_threads())
    t_gen = time.perf_counter() - t_gen
    comp_words = sum(s.size for s in streams)
    flat = torch.empty(comp_words + 2 * n, dtype=torch.int64, pin_memory=True)
    offs = []
    o = 0
    fnp = flat.numpy().view(np.uint64)
    for s in streams:
        fnp[o:o + s.size] = s
        offs.append((o, s.size))
        o += s.size + (s.size & 1)
    dflat = flat.to(dev)
    dstreams = [bq.DeviceRleBitmap(dflat[a:a + b] if b else dflat[:0], r, b) for a, b in offs]
    torch.cuda.synchronize()
    nw = r // 64
    comp_bytes = comp_words * 8
    # N > 1: every rank holds the whole streams and decodes its 1024-aligned word range
    from paper_1402_4073_b200.shard import shard_range
    w0, w1 = shard_range(nw, ctx.world, ctx.rank, 1024)
    out_words = w1 - w0
    # load the RLE kernels once (CUDA loads a module at its first launch) on a small query
    small = _markov_streams(lib, 8, 1 << 16, m1, 600.0, 1)
    wq = bq.RleQuery([bq.DeviceRleBitmap(torch.from_numpy(x.view(np.int64)).to(dev), 1 << 16, x.size)
                      for x in small], 1 << 16)
    for _ in range(2):
        wq.threshold(2)
    torch.cuda.synchronize()
    wq.close()
    out = torch.empty(max(out_words, 1), dtype=torch.int64, device=dev)
    pc = torch.zeros(1, dtype=torch.int64, device=dev)

    # --- fresh queries: K3 directory + first evaluation (K4), CUDA events --------------
    def ev():
        return torch.cuda.Event(enable_timing=True)

    fresh = max(3, min(args.steps, 12))
    offs_np = np.asarray([a for a, _ in offs], dtype=np.uint64)
    lens_np = np.asarray([b for _, b in offs], dtype=np.uint64)
    k3_ms, k4_ms, fresh_ms = [], [], []
    prev = os.environ.get("BQ_RLE_SLICED")
    os.environ["BQ_RLE_SLICED"] = "2"  # the default policy: the first evaluation reads the streams (K4)
    try:
        for i in range(args.warmup + fresh):
            e0, e1, e2 = ev(), ev(), ev()
            torch.cuda.synchronize()
            e0.record(stream)
            # synchronous: K3 on the legacy stream; the packed-streams constructor (one device
            # buffer + offsets) has no per-stream Python marshalling
            qf = bq.RleQuery.from_packed(dflat, offs_np, lens_np, r, word_range=(w0, w1))
            e1.record(stream)
            pc.zero_()
            qf.threshold(t, out, pc, stream=stream)
            e2.record(stream)
            torch.cuda.synchronize()
            if i >= args.warmup:
                k3_ms.append(e0.elapsed_time(e1))
                k4_ms.append(e1.elapsed_time(e2))
                fresh_ms.append(e0.elapsed_time(e2))
            if i + 1 < args.warmup + fresh:
                qf.close()
    finally:
        if prev is None:
            os.environ.pop("BQ_RLE_SLICED", None)
        else:
            os.environ["BQ_RLE_SLICED"] = prev
    q = qf
    fresh_pc = int(pc.item())
    # the same K3 through the list-of-bitmap-objects constructor (per-stream marshalling)
    obj_ms = []
    for _ in range(3):
        e0, e1 = ev(), ev()
        torch.cuda.synchronize()
        e0.record(stream)
        qo = bq.RleQuery(dstreams, r, word_range=(w0, w1))
        e1.record(stream)
        torch.cuda.synchronize()
        obj_ms.append(e0.elapsed_time(e1))
        qo.close()

    # --- repeated queries on the same query object: K4s over the tile-sliced layout -----
    torch.cuda.synchronize()
    t_b = time.perf_counter()
    q.threshold(t, out, pc, stream=stream)  # the second evaluation builds the layout
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_b
    ms_s = _timed_launches(torch, lambda: q.threshold(t, out, pc, stream=stream), args.steps, args.warmup, stream)
    pc.zero_()
    q.threshold(t, out, pc, stream=stream)
    n_mk, n_lit = q.layout_stats
    n_ev = q.layout_events
    tiles = (out_words + 1023) // 1024
    moved = n_ev // 12 * 16 + tiles * 76 + out_words * 8
    mean_s = statistics.mean(ms_s)
    peak, _ = measured_peak()

    # one-shot end to end through the public API from pinned host memory: upload the
    # compressed streams, build the query (K3), one evaluation (K4), result words back
    e2e_line = None
    if not args.no_e2e and ctx.world == 1:
        host_out = torch.empty(max(out_words, 1), dtype=torch.int64, pin_memory=True)
        e2e_s = []
        for _ in range(6):
            torch.cuda.synchronize()
            t_e = time.perf_counter()
            d2 = flat.to(dev, non_blocking=True)
            ds2 = [bq.DeviceRleBitmap(d2[a:a + b] if b else d2[:0], r, b) for a, b in offs]
            q2 = bq.RleQuery(ds2, r)
            o2, p2 = q2.threshold(t)
            host_out.copy_(o2[: q2.out_words], non_blocking=True)
            p2_host = int(p2.item())
            torch.cuda.synchronize()
            e2e_s.append(time.perf_counter() - t_e)
            q2.close()
            del d2, ds2, o2
        e2e_best = statistics.median(e2e_s[1:])
        e2e_line = {"value": round(comp_bytes / e2e_best / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": comp_bytes, "d2h_bytes_per_step": out_words * 8 + 8,
                    "ms_per_step": round(e2e_best * 1e3, 3), "steps": len(e2e_s) - 1,
                    "api": "torch pinned H2D -> engine.RleQuery (bq_rle_query_create: K3) -> threshold (K4) -> D2H",
                    "matches_device_result": bool(p2_host == fresh_pc)}
    from oracle import oracle as O
    # parity on a window: the first 2^26 bits of every stream (the generator is sequential, so a
    # run with r = 2^26 reproduces exactly the prefix of the full stream); rank 0 holds it.  The
    # same window is the CPU baseline's sample (~1-2 s of the single-threaded cdom sweep).
    wr = min(1 << 26, out_words * 64) if ctx.rank == 0 else 1 << 12
    wstreams = _oracle_markov_streams(n, wr, m1, m0, host_threads())
    t0 = time.perf_counter()
    wexp = O.cdom_threshold(wstreams, wr, t)
    cpu_s = time.perf_counter() - t0
    exact_window = ctx.rank != 0 or np.array_equal(out[: wr // 64].cpu().numpy().view(np.uint64), wexp)
    wbytes = sum(s.size for s in wstreams) * 8
    fresh_mean = statistics.mean(fresh_ms)
    # the fresh query must read every stream word and write the result: that is its roofline
    fresh_bytes = int(comp_bytes * out_words / nw) + out_words * 8
    line = _line("c4", comp_bytes * out_words / nw / (fresh_mean / 1e3) / 1e9, fresh_ms, fresh_bytes, len(fresh_ms),
                 args.warmup,
                 {"workload": "C4: N=1024 RLE (EWAH-style) bitmaps, r=2^30 bits, Markov runs (ones mean 256, zeros "
                              f"mean 12544 bits; density 0.02), T={t}; output uncompressed. One step = one FRESH query "
                              "over device-resident streams: K3 directory (bq_rle_query_create) + first evaluation "
                              "(K4 reads the streams); CUDA events around both; streams (2.4 GB) > L2",
                  "n_bitmaps": n, "r_bits": r, "t": t, "compressed_bytes": comp_bytes,
                  "uncompressed_equivalent_bytes": n * nw * 8,
                  "parallelism": f"word-range shards x{ctx.world}, streams replicated" if ctx.world > 1 else "1 GPU"},
                 {"value_note": "EWAH input bytes / fresh-query time (K3 + K4); roofline bytes = the streams once "
                                "+ the uncompressed result",
                  "fresh_query_ms": {"k3_directory": round(statistics.mean(k3_ms), 4),
                                     "k4_first_eval": round(statistics.mean(k4_ms), 4),
                                     "total": round(fresh_mean, 4),
                                     "k3_via_bitmap_objects": round(statistics.median(obj_ms), 4),
                                     "note": "k3 = RleQuery.from_packed (host setup + directory kernel + validation "
                                             "read-back); k3_via_bitmap_objects = RleQuery(list of DeviceRleBitmap)"},
                  "popcount": fresh_pc, "directory_bytes": q.directory_bytes, "host_generation_s": round(t_gen, 2),
                  "repeated_query": {
                      "mean_launch_ms": round(mean_s, 5),
                      "kernel": "K4s over the tile-sliced layout (derived once per query from the streams)",
                      "moved_bytes_per_launch": moved,
                      "moved_gbs": round(moved / (mean_s / 1e3) / 1e9, 1),
                      "moved_frac_of_peak": round(moved / (mean_s / 1e3) / 1e9 / peak, 4),
                      "layout_build_s": round(build_s, 4),
                      "amortized_ms_over_10_queries": round((build_s * 1e3 + 10 * mean_s) / 10, 4),
                      "ewah_bytes_per_query_time_gbs": round(comp_bytes * out_words / nw / (mean_s / 1e3) / 1e9, 1),
                      "note": "not an input-bandwidth figure: K4s does not read the EWAH streams",
                      "layout": {"markers": n_mk, "literal_words": n_lit, "events": n_ev}},
                  "e2e": e2e_line,
                  "matches_oracle_window": bool(exact_window),
                  "cpu_baseline": {"value": round(wbytes / cpu_s / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "port",
                                   "sample": "oracle cdom_threshold (runmerge.py heap sweep restated in C, single "
                                             f"thread as the reference) on the first 2^{wr.bit_length() - 1} bits of all 1024 streams "
                                             f"({wbytes} compressed bytes, {cpu_s:.2f} s)"}},
                 traffic_key="c4_fresh")
    line["gpu_launches"] = len(fresh_ms) * 3  # per fresh query: K3 directory, K4 (phases A, B), K4c (phase C)
    line["_rank_bytes"] = comp_bytes * out_words / nw  # this rank's share of the query
    line["_scaling"] = "strong"
    q.close()
    return line


def run_c5(args, torch, bq, lib, dev, stream, ctx):
    """Config 5: N=511, r=2^32, p=0.5, T=256 (256 GiB), sharded by word range over the
    ranks (8 GPUs: 32 GiB each) with the popcount all-reduced per query.  A rank's
    shard is processed as generate -> compute waves of at most 2^23 words (32 GiB), so
    one GPU runs the whole query as 8 waves; only the query kernels (and the
    all-reduce) are timed."""
    from paper_1402_4073_b200.shard import shard_range

    n, total, t = 511, 1 << 26, 256
    b, e = shard_range(total, ctx.world, ctx.rank)
    wave = min(1 << 23, max(e - b, 1))
    pitch = wave + args.pad_words
    data = torch.empty((n, pitch), dtype=torch.int64, device=dev)
    qarr = np.full(n, 32768, dtype=np.uint32)
    out = torch.empty(wave, dtype=torch.int64, device=dev)
    pc = torch.zeros(1, dtype=torch.int64, device=dev)
    ms_all, rank_ms, pc_total = [], 0.0, 0
    steps = max(1, args.steps // 10)

    def launch(q):
        q.threshold(t, out, pc, stream=stream)
        if ctx.world > 1:
            ctx.dist.all_reduce(pc)

    for w0 in range(b, e, wave):
        wl = min(wave, e - w0)
        _lib_check(lib.bq_gen_bernoulli_rows(SEED, 0, n, qarr.ctypes.data, w0, wl, data.data_ptr(), pitch,
                                             stream.cuda_stream))
        q = bq.ThresholdQuery([data[i, :wl] for i in range(n)], 64 * wl)
        ms = _timed_launches(torch, lambda: launch(q), steps, 1 if w0 > b else args.warmup, stream)
        ms_all += ms
        rank_ms += statistics.mean(ms)
        pc.zero_()
        q.threshold(t, out, pc, stream=stream)
        pc_total += int(pc.item())
        q.close()
    in_bytes_wave = n * wave * 8
    per = statistics.mean(ms_all)
    line = _line("c5", in_bytes_wave / (per / 1e3) / 1e9, ms_all, in_bytes_wave + wave * 8, len(ms_all),
                 args.warmup,
                 {"workload": "C5: N=511, r=2^32 bits, p=0.5, T=256 (256 GiB), word-range shards over the GPUs, each "
                              "processed as generate->compute waves of <= 2^23 words (32 GiB, one GPU's shard at 8 "
                              "GPUs); kernels (+ popcount all-reduce) timed only",
                  "n_bitmaps": n, "r_bits": 64 * total, "t": t, "wave_words": wave,
                  "waves_per_rank": (e - b + wave - 1) // wave,
                  "parallelism": f"word-range shards x{ctx.world}" if ctx.world > 1 else "1 GPU, 8 waves"},
                 {"full_query_ms": round(rank_ms, 3), "popcount": pc_total})
    line["_rank_bytes"] = n * (e - b) * 8
    line["_rank_ms"] = rank_ms
    line["_scaling"] = "strong"
    return line


def run_frows(args, torch, bq, lib, dev, stream, ctx):
    """SURVEY §8(f) rows, each timed with CUDA events after an L2 flush (inputs are
    read from HBM), with its algorithmic bytes:

    * set algebra (f2): bq_binary_op AND / OR / XOR / ANDNOT of two C2 bitmaps
      (2^28 bits: 32 MiB each) and NOT of one;
    * the canonical RLE encoder (f1, K7): the C2 T=16 result (2^28 bits, mixed) and a
      dense Bernoulli(0.5) 2^28-bit bitmap (all literals);
    * an NVRTC-compiled straight-line program (f3): CircuitLibrary(64, 'sideways')
      .program(64, 32) (SSum, majority) over the C2 inputs, next to the counting
      kernel on the same query;
    * the drop-in path (b): api.scan_count on the reference's own UncompressedBitmap
      objects at C1 (host lists in, host list out), next to the reference's own
      scan_count and its fastest algorithm on the same objects."""
    from paper_1402_4073_b200 import api

    n, nw = C2_N, C2_WORDS
    qs = [lib.bq_gen_density_q16(SEED, i, DENS_LO, DENS_HI) for i in range(n)]
    data = torch.empty((n, nw), dtype=torch.int64, device=dev)
    qarr = np.asarray(qs, dtype=np.uint32)
    _lib_check(lib.bq_gen_bernoulli_rows(SEED, 0, n, qarr.ctypes.data, 0, nw, data.data_ptr(), nw,
                                         stream.cuda_stream))
    out = torch.empty(nw, dtype=torch.int64, device=dev)
    pc = torch.zeros(1, dtype=torch.int64, device=dev)
    lnz = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: _l2_flush(scratch)  # noqa: E731
    peak, _ = measured_peak()
    steps = max(5, min(args.steps, 50))
    res = {}

    def rec(name, ms, nbytes, extra=None):
        m = statistics.median(ms)
        d = {"median_ms": round(m, 5), "algorithmic_bytes": int(nbytes),
             "gbs": round(nbytes / (m / 1e3) / 1e9, 1), "frac_of_peak": round(nbytes / (m / 1e3) / 1e9 / peak, 4)}
        if extra:
            d.update(extra)
        res[name] = d

    a, b = data[0], data[1]
    for kind, name in ((0, "and"), (1, "or"), (2, "xor"), (3, "andnot"), (4, "not")):
        def launch(kind=kind):
            _lib_check(lib.bq_binary_op(kind, a.data_ptr(), nw, b.data_ptr(), nw, 64 * nw, out.data_ptr(),
                                        pc.data_ptr(), lnz.data_ptr(), stream.cuda_stream))
        ms = _timed_launches(torch, launch, steps, args.warmup, stream, flush=flush)
        rec(f"binop_{name}", ms, (1 if kind == 4 else 2) * nw * 8 + nw * 8,
            {"kernel": "bq::binop_kernel (128-bit streaming loads)"})
    # the same on operands larger than L2 (8 C2 bitmaps each: 2^25 words = 256 MiB), where
    # launch ramp and tail no longer dominate
    big_a, big_b = data[0:8].reshape(-1), data[8:16].reshape(-1)
    big_out = torch.empty(8 * nw, dtype=torch.int64, device=dev)
    for kind, name in ((0, "and"), (1, "or"), (4, "not")):
        def launch(kind=kind):
            _lib_check(lib.bq_binary_op(kind, big_a.data_ptr(), 8 * nw, big_b.data_ptr(), 8 * nw, 64 * 8 * nw,
                                        big_out.data_ptr(), pc.data_ptr(), lnz.data_ptr(), stream.cuda_stream))
        ms = _timed_launches(torch, launch, steps, args.warmup, stream, flush=flush)
        rec(f"binop_{name}_256mib", ms, ((1 if kind == 4 else 2) + 1) * 8 * nw * 8)
    del big_out
    # exactness of the device set algebra on these operands
    ref_and = (a & b)
    _lib_check(lib.bq_binary_op(0, a.data_ptr(), nw, b.data_ptr(), nw, 64 * nw, out.data_ptr(), pc.data_ptr(),
                                lnz.data_ptr(), stream.cuda_stream))
    res["binop_matches_torch"] = bool(torch.equal(out, ref_and))

    # K7 encoder on the C2 T=16 result and on a dense random bitmap
    query = bq.ThresholdQuery([data[i] for i in range(n)], 64 * nw)
    t16 = torch.empty(nw, dtype=torch.int64, device=dev)
    query.threshold(16, t16, pc, stream=stream)
    dense = torch.empty((1, nw), dtype=torch.int64, device=dev)
    q05 = np.asarray([32768], dtype=np.uint32)
    _lib_check(lib.bq_gen_bernoulli_rows(SEED + 1, 0, 1, q05.ctypes.data, 0, nw, dense.data_ptr(), nw,
                                         stream.cuda_stream))
    import ctypes
    enc = torch.empty(nw + 2, dtype=torch.int64, device=dev)
    for name, src in (("encode_c2_t16_result", t16), ("encode_dense", dense[0])):
        n_out = ctypes.c_uint64(0)

        def launch(src=src, n_out=n_out):
            _lib_check(lib.bq_rle_encode_device(src.data_ptr(), nw, 64 * nw, enc.data_ptr(), nw + 2,
                                                ctypes.byref(n_out), stream.cuda_stream))
        ms = _timed_launches(torch, launch, max(5, steps // 2), args.warmup, stream, flush=flush)
        rec(name, ms, nw * 8 + int(n_out.value) * 8,
            {"encoded_words": int(n_out.value), "kernel": "K7 (classify / CUB select / size / CUB scan / scatter)",
             "note": "synchronous call: includes its host round trips"})
    host_enc = enc[: int(n_out.value)].cpu().numpy().view(np.uint64)
    from oracle import oracle as O
    res["encode_matches_oracle"] = bool(np.array_equal(host_enc, O.rle_compress(dense[0].cpu().numpy().view(np.uint64),
                                                                                64 * nw)))

    # NVRTC SSum(64, 32) program over the C2 inputs, and the counting kernel on the same query
    lib_c = api.CircuitLibrary(n_max=64, builder="sideways")
    prog = api.compile_program(lib_c.program(64, 32))

    def launch_prog():
        prog.run(query, out, pc, lnz, stream=stream)
    ms = _timed_launches(torch, launch_prog, steps, args.warmup, stream, flush=flush)
    rec("nvrtc_ssum_64_32", ms, n * nw * 8 + nw * 8, {"gates": lib_c.program(64, 32).op_count,
                                                        "kernel": "bq_prog (NVRTC, sm_100a)"})
    prog_out = out.clone()
    ms = _timed_launches(torch, lambda: query.threshold(32, out, pc, stream=stream), steps, args.warmup, stream,
                         flush=flush)
    rec("count_kernel_t32_same_query", ms, n * nw * 8 + nw * 8)
    res["nvrtc_matches_count_kernel"] = bool(torch.equal(prog_out, out))
    query.close()
    del data, dense, scratch
    torch.cuda.empty_cache()

    # drop-in e2e at C1 through api.scan_count on the reference's own objects
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "bitquorum")):
        sys.path.insert(0, ref_dir)
        from bitquorum import bitmaps as rbm
        from bitquorum import counters
        from bitquorum.circuits import csv_threshold

        n1, nw1, t1 = 8, 1 << 14, 3
        ins = [rbm.UncompressedBitmap([int(w) for w in O.gen_bernoulli(SEED, i, 6554, 0, nw1)], 64 * nw1)
               for i in range(n1)]
        api.scan_count(ins, t1)  # warm: upload cache and query cache hold these objects afterwards
        times = []
        for _ in range(5):
            # fresh objects each time: the full drop-in cost (upload, query, download, list result)
            fresh = [rbm.UncompressedBitmap(list(b.words), b.bit_length) for b in ins]
            t0 = time.perf_counter()
            got = api.scan_count(fresh, t1)
            times.append(time.perf_counter() - t0)
        cached = []
        for _ in range(5):
            t0 = time.perf_counter()
            api.scan_count(ins, t1)
            cached.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        exp = counters.scan_count(ins, t1)
        ref_sc = time.perf_counter() - t0
        t0 = time.perf_counter()
        csv_threshold(ins, t1)
        ref_csv = time.perf_counter() - t0
        nbytes = n1 * nw1 * 8
        res["drop_in_c1"] = {
            "api": "paper_1402_4073_b200.scan_count(reference UncompressedBitmap objects)",
            "fresh_objects_ms": round(statistics.median(times) * 1e3, 3),
            "fresh_objects_gbs": round(nbytes / statistics.median(times) / 1e9, 4),
            "cached_objects_ms": round(statistics.median(cached) * 1e3, 3),
            "reference_scan_count_ms": round(ref_sc * 1e3, 1),
            "reference_csv_threshold_ms": round(ref_csv * 1e3, 1),
            "matches_reference": bool(got == exp),
            "note": "host lists in, host list out: upload, query, download and the list result inside the "
                    "timing; cached = the same objects again (upload and query caches hit)"}
    line = {"metric": METRIC, "workload": "frows", "unit": "GB/s", "n_gpus": 1, "steps": steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": "u64", "data": "synthetic (seed 1402)",
            "config": {"workload": "SURVEY §8(f) rows and the drop-in path, each timed after a 256 MB L2 flush"},
            "rows": res}
    big = res["binop_and_256mib"]
    line["value"] = big["gbs"]
    line["roofline"] = {"bound": "hbm", "achieved": big["gbs"], "peak": peak, "unit": "GB/s",
                        "frac": big["frac_of_peak"], "kernel": "bq::binop_kernel (AND, 256 MiB operands)",
                        "traffic": ncu_traffic("binop"),
                        "algorithmic_bytes_per_launch": big["algorithmic_bytes"],
                        "mean_launch_ms": big["median_ms"]}
    line["ms_per_step"] = big["median_ms"]
    line["gpu_launches"] = 8 * steps
    line["_rank_bytes"] = big["algorithmic_bytes"]
    line["_rank_ms"] = big["median_ms"]
    return line


def _lib_check(rc):
    from paper_1402_4073_b200 import _lib
    _lib.check(rc)


def run_extra(args):
    """Workloads c1/c3/c4/c5.  Under torchrun (N > 1): c4 and c5 shard the query by word
    range (strong scaling); c1 and c3 run one replica per GPU (weak scaling).  The
    job's value is the bytes all ranks processed over the slowest rank's time."""
    import types

    import torch
    import torch.distributed as dist

    import paper_1402_4073_b200 as bq
    from paper_1402_4073_b200 import _lib

    rank, world, local = _dist_setup(torch, dist)
    lib = _lib.load()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    ctx = types.SimpleNamespace(world=world, rank=rank, dist=dist, cpu=(world == 1))
    fn = {"c1": run_c1, "c3": run_c3, "c4": run_c4, "c5": run_c5, "frows": run_frows}[args.workload]
    with ClockSampler(physical_gpu_index(local)) as clocks:
        line = fn(args, torch, bq, lib, dev, stream, ctx)
    rank_bytes = float(line.pop("_rank_bytes", line["roofline"]["algorithmic_bytes_per_launch"]))
    rank_ms = float(line.pop("_rank_ms", line["roofline"]["mean_launch_ms"]))
    scaling = line.pop("_scaling", "weak")
    if world > 1:
        red = torch.tensor([rank_ms, rank_bytes, float(line.get("popcount", 0))], dtype=torch.float64, device=dev)
        mx = red.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(red, op=dist.ReduceOp.SUM)
        job_ms, job_bytes = float(mx[0]), float(red[1])
        line["n_gpus"] = world
        line["scaling"] = scaling
        line["value"] = round(job_bytes / (job_ms / 1e3) / 1e9, 3)
        line["ms_per_step"] = round(job_ms, 5)
        if "popcount" in line and args.workload in ("c4", "c5"):
            line["popcount"] = int(red[2])  # shards: the whole result's popcount
        line.pop("cpu_baseline", None)  # CPU baseline: rank 0 at N=1 only
    line["clocks"] = clocks.summary()
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def self_launch(n: int) -> int:
    """``--gpus N`` outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and the same arguments; rank 0 prints the
    line.  The ranks need N visible GPUs (or BQ_BENCH_SHARE_GPU=1, a functional
    check that is not a measurement)."""
    import socket

    if os.environ.get("BQ_BENCH_SHARE_GPU") != "1":
        import torch

        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--workload", choices=("c1", "c2", "c3", "c4", "c5", "frows"), default="c2",
                    help="BASELINE config; c2 (the default) is the headline line")
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--pad-words", type=int, default=256, help="row pitch padding (words) between bitmaps")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunk-mib", type=int, default=0, help="host streaming chunk (MiB of input; 0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reference-python", action="store_true",
                    help="--impl reference: skip timing the stock reference Python (context numbers)")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 strong-scaling fields of the default line")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--c4-t", type=int, default=50, help="C4 threshold (BASELINE configs[3]: 50; others are diagnostics)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return self_launch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "c2":
        return run_extra(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
