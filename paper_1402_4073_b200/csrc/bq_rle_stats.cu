// K8: the reference's cdom introspection counters, computed on the device.
//
// runmerge.cdom_threshold / cdom_symmetric (runmerge.py:198-241, :244-299) fill
// ``stats`` with the counts of their CPU sweep: ``segments`` (sweep steps),
// ``heap_pops`` (runs retired from the heap) and, for thresholds, ``branches``
// (dirty_segment_solver's dispatch: or / and / looped / scan, :69-83).  The
// device path never runs that sweep, but each count is a function of the
// inputs' merged runs (_merged_runs, :29-56), so it is recomputed here from the
// K3 tile directory:
//   heap_pops = the number of merged runs over all inputs (each is popped once);
//   segments  = the number of distinct merged-run end positions (a segment ends
//               exactly where some input's run ends);
//   branches  = per segment [s, e] whose outcome is open (0 < T - k <= d, with
//               k one-fills and d dirty inputs), the solver's choice, which needs
//               beta = the set bits of the dirty inputs' literal words in [s, e].
// Pass 1 (one thread per (tile, stream)) walks the stream's markers across its
// tile from the directory entry and records, at positions inside the tile only:
// run ends (a bitmap, plus a count), the packed one-fill / dirty difference array
// (ones in bits 0-31, dirty inputs in 32-63) and each word's literal popcount.
// Two scans turn those into (k_w, d_w) and prefix popcounts; pass 2 (one thread
// per 64 positions) visits every segment end.  Introspection only: one call,
// synchronous, ~20 B of scratch per output word.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include "bq_internal.h"

namespace bq {

namespace {

constexpr uint64_t kOne = 1ull;
constexpr uint64_t kDirty = 1ull << 32;

struct StatsWalkArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    const uint2 *dir;
    int n;
    uint32_t ntiles;
    uint64_t total;
    unsigned long long *diff;     // [total + 1] packed difference array
    unsigned long long *litpop;   // [total] set bits of literal words at each word
    unsigned long long *ends;     // [ceil(total / 64)] run-end bitmap
    unsigned long long *counters; // [0] heap pops
};

__device__ __forceinline__ void split(uint64_t mk, uint32_t &bit, uint64_t &run, uint64_t &dirty) {
    bit = (uint32_t)(mk & 1);
    run = (mk >> 1) & 0xFFFFFFFFull;
    dirty = mk >> 33;
}

__global__ void __launch_bounds__(256) sweep_walk_kernel(StatsWalkArgs a) {
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pops = 0;
    if (idx < (uint64_t)a.ntiles * a.n) {
        const uint32_t tile = (uint32_t)(idx / (uint64_t)a.n);
        const int st = (int)(idx % (uint64_t)a.n);
        const uint64_t *s = a.ptrs[st];
        const uint64_t L = a.lens[st];
        const uint2 e = a.dir[idx];
        const uint64_t ts = (uint64_t)tile * kRleTile;
        const uint64_t te = min(ts + kRleTile, a.total);
        uint64_t i = e.x, pos = e.y;
        auto mark = [&](uint64_t end) {
            if (end >= ts && end < te) {
                atomicOr(a.ends + (end >> 6), 1ull << (end & 63));
                ++pops;
            }
        };
        while (i < L && pos < te) {
            uint32_t bit;
            uint64_t run, dirty;
            split(__ldg(s + i), bit, run, dirty);
            const uint64_t fe = pos + run, de = fe + dirty;
            if (run | dirty) {
                // an update belongs to the tile of the word it describes: a start or a
                // fill-to-literal change to its own word, a marker's end to its last word
                // (the thread of the tile holding word de is not handed that marker when
                // de is a tile boundary)
                if (bit && run && pos >= ts) atomicAdd(a.diff + pos, kOne);
                if (dirty) {
                    const uint64_t dfe = kDirty - ((bit && run) ? kOne : 0);
                    if (fe >= ts && fe < te) atomicAdd(a.diff + fe, (unsigned long long)dfe);
                    if (de - 1 >= ts && de - 1 < te && de < a.total)
                        atomicAdd(a.diff + de, (unsigned long long)(0 - kDirty));
                } else if (bit && run && fe - 1 >= ts && fe - 1 < te && fe < a.total) {
                    atomicAdd(a.diff + fe, (unsigned long long)(0 - kOne));
                }
                if (dirty) {
                    const uint64_t lo = max(fe, ts), hi = min(de, te);
                    for (uint64_t p = lo; p < hi; ++p)
                        atomicAdd(a.litpop + p, (unsigned long long)__popcll(__ldg(s + i + 1 + (p - fe))));
                    mark(de - 1);  // a literal group is one run of its own
                }
                if (run && fe - 1 >= ts && fe - 1 < te) {
                    // a fill's run ends unless the next segment _merged_runs sees is a fill of
                    // the same bit (the implicit zero tail included); empty markers yield nothing
                    bool ends = dirty != 0;
                    if (!ends) {
                        uint64_t j = i + 1, nm = 0;
                        while (j < L && ((nm = __ldg(s + j)) >> 1) == 0) ++j;  // run == dirty == 0
                        if (j < L) ends = ((nm >> 1) & 0xFFFFFFFFull) == 0 || (uint32_t)(nm & 1) != bit;
                        else ends = !(fe < a.total && bit == 0);
                    }
                    if (ends) mark(fe - 1);
                }
            }
            pos = de;
            i += 1 + dirty;
        }
        if (i >= L && pos < a.total) mark(a.total - 1);  // implicit zero tail (bitmaps.py:218-219)
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pops += __shfl_down_sync(0xffffffffu, pops, o);
    if ((threadIdx.x & 31) == 0 && pops) atomicAdd(a.counters, pops);
}

// highest end position in each 64-word group of the end bitmap, -1 if none
__global__ void last_end_kernel(const unsigned long long *ends, uint64_t nw, long long *last) {
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nw) return;
    const unsigned long long w = ends[j];
    last[j] = w ? (long long)(j * 64 + 63 - __clzll((long long)w)) : -1ll;
}

struct MaxOp {
    __device__ __forceinline__ long long operator()(long long x, long long y) const { return x > y ? x : y; }
};

// counters: [1] segments, [2..5] or / and / looped / scan
__global__ void __launch_bounds__(256) segment_kernel(const unsigned long long *ends, uint64_t nw,
                                                      const long long *last_scan, const unsigned long long *kd,
                                                      const unsigned long long *pre, int t,
                                                      unsigned long long *counters) {
    __shared__ unsigned long long sc[5];
    if (threadIdx.x < 5) sc[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nw) {
        unsigned long long w = ends[j];
        long long prev = j ? last_scan[j - 1] : -1ll;
        unsigned long long c[5] = {0, 0, 0, 0, 0};
        while (w) {
            const int b = __ffsll((long long)w) - 1;
            w &= w - 1;
            const uint64_t e = j * 64 + (uint64_t)b;
            c[0]++;
            if (t > 0) {
                const unsigned long long v = kd[e];
                const int k = (int)(uint32_t)v, d = (int)(v >> 32);
                const int te = t - k;
                if (te > 0 && te <= d) {  // the solver runs (runmerge.py:226-233)
                    int br;
                    if (te == 1) br = 0;
                    else if (te == d) br = 1;
                    else if (te >= 128) br = 3;  // SCANCOUNT_CUTOFF (:25)
                    else {
                        const unsigned long long beta = pre[e] - (prev >= 0 ? pre[prev] : 0ull);
                        br = 2 * beta >= (unsigned long long)d * (unsigned long long)te ? 2 : 3;
                    }
                    c[1 + br]++;
                }
            }
            prev = (long long)e;
        }
        for (int k = 0; k < 5; ++k)
            if (c[k]) atomicAdd(&sc[k], c[k]);
    }
    __syncthreads();
    if (threadIdx.x < 5 && sc[threadIdx.x]) atomicAdd(counters + 1 + threadIdx.x, sc[threadIdx.x]);
}

}  // namespace

int rle_sweep_stats(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const uint2 *d_dir, int n,
                    uint32_t ntiles, uint64_t total, int t, uint64_t *h_stats, cudaStream_t s) {
    const uint64_t nw = (total + 63) / 64;
    size_t t_diff = 0, t_pop = 0, t_max = 0;
    cub::DeviceScan::InclusiveSum(nullptr, t_diff, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                  (int64_t)total, s);
    cub::DeviceScan::InclusiveScan(nullptr, t_max, (long long *)nullptr, (long long *)nullptr, MaxOp(),
                                   (int64_t)nw, s);
    const size_t tmp = std::max(t_diff, t_max);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_diff = al((total + 1) * 8), b_pop = al(total * 8), b_ends = al(nw * 8), b_last = al(nw * 8),
                 b_cnt = al(6 * 8);
    char *mem = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&mem), b_diff + b_pop + b_ends + 2 * b_last + b_cnt + tmp, s);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(sweep stats)");
    (void)t_pop;
    auto *diff = reinterpret_cast<unsigned long long *>(mem);
    auto *litpop = reinterpret_cast<unsigned long long *>(mem + b_diff);
    auto *ends = reinterpret_cast<unsigned long long *>(mem + b_diff + b_pop);
    auto *last = reinterpret_cast<long long *>(mem + b_diff + b_pop + b_ends);
    auto *last_scan = reinterpret_cast<long long *>(mem + b_diff + b_pop + b_ends + b_last);
    auto *cnt = reinterpret_cast<unsigned long long *>(mem + b_diff + b_pop + b_ends + 2 * b_last);
    void *scratch = mem + b_diff + b_pop + b_ends + 2 * b_last + b_cnt;
    e = cudaMemsetAsync(mem, 0, b_diff + b_pop + b_ends, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 6 * 8, s);
    if (e == cudaSuccess) {
        StatsWalkArgs a{d_ptrs, d_lens, d_dir, n, ntiles, total, diff, litpop, ends, cnt};
        const uint64_t threads = (uint64_t)ntiles * n;
        sweep_walk_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a);
        e = cudaGetLastError();
    }
    size_t tb = tmp;
    if (e == cudaSuccess && t > 0) {
        e = cub::DeviceScan::InclusiveSum(scratch, tb, diff, diff, (int64_t)total, s);
        tb = tmp;
        if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(scratch, tb, litpop, litpop, (int64_t)total, s);
    }
    if (e == cudaSuccess) {
        last_end_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(ends, nw, last);
        tb = tmp;
        e = cub::DeviceScan::InclusiveScan(scratch, tb, last, last_scan, MaxOp(), (int64_t)nw, s);
    }
    if (e == cudaSuccess) {
        segment_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(ends, nw, last_scan, diff, litpop, t, cnt);
        e = cudaGetLastError();
    }
    unsigned long long h[6] = {0, 0, 0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(mem, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "sweep stats");
    h_stats[0] = h[1];  // segments
    h_stats[1] = h[0];  // heap pops
    for (int k = 0; k < 4; ++k) h_stats[2 + k] = h[2 + k];
    return BQ_OK;
}

}  // namespace bq
