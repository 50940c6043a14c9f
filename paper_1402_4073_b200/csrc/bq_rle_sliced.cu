// K4 over the tile-sliced RLE layout (see SlicedLayout in bq_internal.h).
//
// The per-stream K4 (bq_rle.cu) gives each lane one stream and follows its
// marker chain: a dependent shared-memory load per marker, and lanes idle while
// the longest chain of the warp finishes (~47% lane efficiency on C4).  Here the
// streams are re-encoded once per query, every 1024-word slice of every stream
// into what K4s reads and nothing more:
//  - for phase A, the nonzero updates the slice's markers make to the tile's
//    difference array (ones | dirty << 16), as 10-bit positions in six per-tile
//    lists by update kind, packed 12 to a 16-byte vector and permuted so that each
//    shared-memory atomic instruction hits 32 distinct banks.  Phase A then costs
//    two ALU instructions and one shared-memory add per event, with a warp-uniform
//    constant -- no field extraction, prefix sums or zero-update redirects (the
//    marker decode it replaces was ALU-pipe bound at ~28 thread instructions per
//    marker);
//  - for phase C, the slice's literal words, position-major per tile, so the
//    literal words of an undecided word are contiguous.  Literal words are read
//    only at undecided positions, as runmerge.cdom_threshold examines dirty words
//    only where the fill counts do not decide (runmerge.py:198-241).
//
// Per tile (one CTA, tiles in descending order of reach): A) events staged into
// shared memory by TMA bulk copies in 10 KB pieces (double-buffered) and added into
// the packed difference array cnt; B) prefix sum and const_until decisions;
// C) bit-sliced literal counts of undecided words.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "bq_internal.h"
#include "bq_rle_tile.cuh"

namespace bq {

namespace {

#ifndef BQ_SL_NT
#define BQ_SL_NT 128
#define BQ_SL_MINB 8
#endif
constexpr int kSlNT = BQ_SL_NT;                            // K4s threads per CTA (4 warps)
#ifndef BQ_SL_PIECE
#define BQ_SL_PIECE 640
#endif
constexpr int kPieceVecs = BQ_SL_PIECE;                    // event vectors per staged piece (10 KB; 8 CTAs per SM)
constexpr uint32_t kThreadWordMax = 128;                   // phase C: words with more literals get a warp
constexpr int kLitStarts = kRleTile + 1;                   // literal offsets per tile (position-major)
constexpr int kSlCntWords = kRleTile + 4;                  // difference array + sentinel (+ pad)
constexpr size_t kSlBufBytes = 2 * (size_t)kPieceVecs * 16;
constexpr size_t kSlPhaseC = (size_t)kRleTile * 4;  // undecided and heavy word lists
constexpr size_t kSlRegion = kSlBufBytes > kSlPhaseC ? kSlBufBytes : kSlPhaseC;
constexpr size_t kSlSmem = 16 + kSlRegion;  // 2 mbarriers | region (dynamic; the difference array is static)

// ---------------------------------------------------------------------------
// Layout build, one thread per (tile, stream) slice.  The counting pass maps
// neighbouring threads to neighbouring tiles of one stream (their reads are
// adjacent); the emitting pass to neighbouring streams of one tile (their writes
// are adjacent in the tile-major output): 0.9 + 3.0 ms at C4 instead of 0.9 + 5.3.

struct SliceSink {
    uint64_t *lit;           // the slice's first literal word in the tile's literal array
    uint16_t *pos;           // ... and its word position in the parallel array
    uint16_t *ev[kEvKinds];  // the slice's first entry in each of the tile's event lists
};

struct SliceCounts {
    uint32_t mk, lit;
    uint32_t ev[kEvKinds];  // events of each kind (bq_internal.h; deltas in add_vector)
};

// Re-encode stream words [ts, ts + 1024) starting at the directory entry e
// (marker index, fill start): the slice's literal words with their positions, and
// its nonzero updates to the difference array (events at positions inside the tile;
// a literal group's end is merged with what the next marker starts at the same
// position).  Markers are counted (a layout statistic), not stored.
template <bool EMIT>
__device__ SliceCounts slice_walk(const uint64_t *src, uint64_t L, uint2 e, uint64_t ts, const SliceSink &sink) {
    const uint64_t te = ts + kRleTile;
    uint64_t i = e.x, pos = e.y;
    uint32_t rel = 0;
    SliceCounts n{};
    bool pend = false;  // the previous marker's literal group ends at rel (its -1 << 16 not yet filed)
    auto event = [&](int kind, uint32_t at) {
        if (EMIT) sink.ev[kind][n.ev[kind]] = (uint16_t)at;
        ++n.ev[kind];
    };
    auto emit = [&](uint32_t bit, uint32_t run, uint32_t dirty) {
        const uint32_t fe = rel + run, de = fe + dirty;
        if (EMIT)
            for (uint32_t k = 0; k < dirty; ++k) sink.pos[n.lit + k] = (uint16_t)(fe + k);
        bool cancel = false;  // a pending literal end meets this marker's literal start (run 0)
        if (pend) {
            if (bit) event(4, rel);
            else if (run == 0u && dirty) cancel = true;
            else event(3, rel);
        } else if (bit) {
            event(0, rel);
        }
        if (bit) {
            if (dirty) event(5, fe);
            else if (fe < (uint32_t)kRleTile) event(1, fe);
        } else if (dirty && !cancel) {
            event(2, fe);
        }
        pend = dirty && de < (uint32_t)kRleTile;
        ++n.mk;
        rel = de;
    };
    while (rel < (uint32_t)kRleTile) {
        if (i >= L) {  // implicit zero tail
            emit(0u, (uint32_t)kRleTile - rel, 0u);
            break;
        }
        const uint64_t m = __ldg(src + i);
        const uint64_t run = (m >> 1) & 0xFFFFFFFFull, dirty = m >> 33;
        const uint64_t fe = pos + run, de = fe + dirty;
        const uint64_t cfs = max(pos, ts), cfe = min(fe, te);
        const uint64_t cds = max(fe, ts), cde = min(de, te);
        const uint32_t crun = cfe > cfs ? (uint32_t)(cfe - cfs) : 0u;
        const uint32_t cdirty = cde > cds ? (uint32_t)(cde - cds) : 0u;
        if (crun + cdirty) {
            if (EMIT)
                for (uint32_t k = 0; k < cdirty; ++k) sink.lit[n.lit + k] = __ldg(src + i + 1 + (cds - fe) + k);
            emit((uint32_t)(m & 1) & (crun != 0u), crun, cdirty);
            n.lit += cdirty;
        }
        pos = de;
        i += 1 + dirty;
    }
    return n;
}

__global__ void slice_count_kernel(const uint64_t *const *ptrs, const uint64_t *lens, const uint2 *dir, int n,
                                   uint32_t tile0, uint32_t ntiles, uint64_t *counts, ulonglong4 *ecounts) {
    const uint64_t total = (uint64_t)ntiles * n;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const int s = (int)(k / ntiles);  // neighbouring threads: neighbouring tiles of one stream (reads)
        const uint32_t t = (uint32_t)(k % ntiles);
        const SliceCounts c =
            slice_walk<false>(ptrs[s], lens[s], dir[(size_t)t * n + s], (uint64_t)(tile0 + t) * kRleTile, SliceSink{});
        counts[(size_t)t * n + s] = (uint64_t)c.mk | ((uint64_t)c.lit << 32);
        ecounts[(size_t)t * n + s] = make_ulonglong4((uint64_t)c.ev[0] | ((uint64_t)c.ev[1] << 32),
                                                     (uint64_t)c.ev[2] | ((uint64_t)c.ev[3] << 32),
                                                     (uint64_t)c.ev[4] | ((uint64_t)c.ev[5] << 32), 0ull);
    }
}

// One CTA per tile: exclusive scans of the slice counts in place (two 32-bit counts
// per 64-bit value: each half of a tile's sum stays below 2^32), and the tile totals:
// markers, literals, the tile's list descriptor (cumulative list ends in 16-byte
// vectors, each list padded to whole warp rows, and the lists' real lengths) and
// the tile's vector total.
__global__ void __launch_bounds__(1024) slice_scan_kernel(uint64_t *counts, ulonglong4 *ecounts, int n, uint64_t *tile_m,
                                                          uint64_t *tile_l, uint64_t *tile_e, uint4 *desc) {
    using Scan = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint64_t carry[4];
    const uint32_t t = blockIdx.x;
    uint64_t *row = counts + (size_t)t * n;
    ulonglong4 *erow = ecounts + (size_t)t * n;
    if (threadIdx.x < 4) carry[threadIdx.x] = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int s = base + (int)threadIdx.x;
        const ulonglong4 ev = s < n ? erow[s] : make_ulonglong4(0ull, 0ull, 0ull, 0ull);
        const uint64_t v[4] = {s < n ? row[s] : 0ull, ev.x, ev.y, ev.z};
        uint64_t ex[4], agg[4], c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q) __syncthreads();
            Scan(tmp).ExclusiveSum(v[q], ex[q], agg[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = carry[q];
        if (s < n) {
            row[s] = ex[0] + c[0];
            erow[s] = make_ulonglong4(ex[1] + c[1], ex[2] + c[2], ex[3] + c[3], 0ull);
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int q = 0; q < 4; ++q) carry[q] = c[q] + agg[q];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint64_t m = carry[0] & 0xFFFFFFFFull, l = carry[0] >> 32;
        tile_m[t] = m;
        tile_l[t] = l;
        uint32_t end[kEvKinds], real[kEvKinds], acc = 0;
        for (int k = 0; k < kEvKinds; ++k) {
            real[k] = (uint32_t)(carry[1 + k / 2] >> (32 * (k & 1)));
            acc += (real[k] + kEvRow - 1) / kEvRow * 32;
            end[k] = acc;
        }
        desc[3 * (size_t)t] = make_uint4(end[0], end[1], end[2], end[3]);
        desc[3 * (size_t)t + 1] = make_uint4(end[4], end[5], real[0], real[1]);
        desc[3 * (size_t)t + 2] = make_uint4(real[2], real[3], real[4], real[5]);
        tile_e[t] = acc;
    }
}

__global__ void slice_emit_kernel(const uint64_t *const *ptrs, const uint64_t *lens, const uint2 *dir, int n,
                                  uint32_t tile0, uint32_t ntiles, const uint64_t *offs, const ulonglong4 *eoffs,
                                  const uint64_t *lbase, const uint64_t *ebase, const uint4 *desc,
                                  uint64_t *literals, uint16_t *lit_pos, uint16_t *events) {
    const uint64_t total = (uint64_t)ntiles * n;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const int s = (int)(k % n);  // neighbouring threads: neighbouring slices of one tile (writes)
        const uint32_t t = (uint32_t)(k / n);
        const uint64_t o = offs[(size_t)t * n + s];
        const ulonglong4 eo = eoffs[(size_t)t * n + s];
        const uint4 ea = desc[3 * (size_t)t], eb = desc[3 * (size_t)t + 1];
        const uint32_t starts[kEvKinds] = {0u, ea.x, ea.y, ea.z, ea.w, eb.x};
        const uint32_t within[kEvKinds] = {(uint32_t)eo.x, (uint32_t)(eo.x >> 32), (uint32_t)eo.y,
                                           (uint32_t)(eo.y >> 32), (uint32_t)eo.z, (uint32_t)(eo.z >> 32)};
        uint16_t *tev = events + ebase[t] * kEvVec;  // positions as emitted: one 16-bit slot per event
        SliceSink sink;
        sink.lit = literals + lbase[t] + (uint32_t)(o >> 32);
        sink.pos = lit_pos + lbase[t] + (uint32_t)(o >> 32);
#pragma unroll
        for (int q = 0; q < kEvKinds; ++q) sink.ev[q] = tev + (size_t)starts[q] * kEvVec + within[q];
        slice_walk<true>(ptrs[s], lens[s], dir[(size_t)t * n + s], (uint64_t)(tile0 + t) * kRleTile, sink);
    }
}

__global__ void gather_meta_kernel(const uint32_t *order, const uint4 *desc, const uint64_t *ebase, TileMeta *meta,
                                   uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = order[i];
    TileMeta tm;
    tm.desc[0] = desc[3 * (size_t)t];
    tm.desc[1] = desc[3 * (size_t)t + 1];
    tm.desc[2] = desc[3 * (size_t)t + 2];
    tm.ebase = ebase[t];
    tm.tile = t;
    tm.pad = 0;
    meta[i] = tm;
}

__global__ void iota_kernel(uint32_t *ids, uint32_t n) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) ids[k] = k;
}

// One CTA per tile: the tile's literal words (emitted slice by slice, each with its
// word position) reordered position-major -- the literals at word p of the tile are
// [lit_start[p], lit_start[p + 1]) -- by a counting sort over the 1024 positions.
__global__ void __launch_bounds__(512) sort_literals_kernel(const uint64_t *lit_src, const uint16_t *pos_src,
                                                            const uint64_t *lbase, uint64_t *lit, uint32_t *lit_start) {
    using Scan = cub::BlockScan<uint32_t, 512>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t start[kRleTile], fill[kRleTile];
    const uint32_t t = blockIdx.x;
    const int tid = threadIdx.x;
    const uint64_t b = lbase[t];
    const uint32_t n = (uint32_t)(lbase[t + 1] - b);
    for (int k = tid; k < kRleTile; k += 512) {
        start[k] = 0;
        fill[k] = 0;
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += 512) atomicAdd(&start[pos_src[b + i]], 1u);
    __syncthreads();
    const uint32_t v0 = start[2 * tid], v1 = start[2 * tid + 1];
    uint32_t ex;
    Scan(tmp).ExclusiveSum(v0 + v1, ex);
    __syncthreads();
    start[2 * tid] = ex;
    start[2 * tid + 1] = ex + v0;
    uint32_t *ls = lit_start + (size_t)t * kLitStarts;
    ls[2 * tid] = ex;
    ls[2 * tid + 1] = ex + v0;
    if (tid == 0) ls[kRleTile] = n;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += 512) {
        const uint32_t p = pos_src[b + i];
        lit[b + start[p] + atomicAdd(&fill[p], 1u)] = lit_src[b + i];
    }
}

// One CTA per (tile, event kind): permute the list (emitted slice by slice) so that
// each shared-memory atomic instruction of phase A -- event j of the 32 vectors of a
// warp row -- updates 32 distinct banks, and pack it.  Events are ranked within their
// bank (bank = position mod 32), ordered by (rank, bank) -- every round of ranks holds
// each bank at most once -- and position s of that order becomes event j =
// (s mod kEvRow) / 32 of vector (s / kEvRow) * 32 + s mod 32 of the list: 10-bit field
// j mod 3 of 32-bit word j / 3.  Groups of 32 spanning two rounds can repeat a bank
// once.  Ranks follow list order (deterministic layout).  Slots past the list's real
// length stay zero; phase A skips them.  dst is zeroed beforehand.
__global__ void __launch_bounds__(256) arrange_events_kernel(const uint16_t *src, uint32_t *dst, const uint64_t *ebase,
                                                             const uint4 *desc) {
    const uint32_t t = blockIdx.x, kind = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint4 ea = desc[3 * (size_t)t], eb = desc[3 * (size_t)t + 1], ec = desc[3 * (size_t)t + 2];
    const uint32_t ends[kEvKinds] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y};
    const uint32_t reals[kEvKinds] = {eb.z, eb.w, ec.x, ec.y, ec.z, ec.w};
    const uint32_t vstart = kind ? ends[kind - 1] : 0u;
    const uint32_t nreal = reals[kind];
    const uint64_t vbase = ebase[t] + vstart;
    const uint16_t *s = src + vbase * kEvVec;
    uint32_t *d = dst + vbase * 4;
    __shared__ uint32_t bank_cnt[32], running[32], wcnt[8][32];
    __shared__ uint32_t sorted_cnt[32], sorted_bank[32], prefix[33], sufmask[33];
    auto place = [&](uint32_t sidx, uint32_t pos) {
        const uint32_t within = sidx % kEvRow, j = within / 32;
        const uint32_t vec = sidx / kEvRow * 32 + within % 32;
        atomicOr(d + (size_t)vec * 4 + j / 3, pos << (10 * (j % 3) + 2));  // byte offsets: bits 2-11, 12-21, 22-31
    };
    if (tid < 32) {
        bank_cnt[tid] = 0;
        running[tid] = 0;
    }
    __syncthreads();
    for (uint32_t i = tid; i < nreal; i += 256) atomicAdd(&bank_cnt[s[i] & 31u], 1u);
    __syncthreads();
    if (tid < 32) {  // banks ordered by (count, bank)
        const uint32_t c = bank_cnt[tid];
        uint32_t pos = 0;
        for (int b = 0; b < 32; ++b) {
            const uint32_t cb = bank_cnt[b];
            pos += (cb < c || (cb == c && b < tid)) ? 1u : 0u;
        }
        sorted_cnt[pos] = c;
        sorted_bank[pos] = (uint32_t)tid;
    }
    __syncthreads();
    if (tid == 0) {
        prefix[0] = 0;
        for (int k = 0; k < 32; ++k) prefix[k + 1] = prefix[k] + sorted_cnt[k];
        sufmask[32] = 0;
        for (int k = 31; k >= 0; --k) sufmask[k] = sufmask[k + 1] | (1u << sorted_bank[k]);
    }
    __syncthreads();
    for (uint32_t c0 = 0; c0 < nreal; c0 += 256) {
        const uint32_t i = c0 + tid;
        const bool valid = i < nreal;
        const uint32_t v = valid ? s[i] : 0u;
        const uint32_t b = v & 31u;
        wcnt[warp][lane] = 0;
        __syncwarp();
        const uint32_t peers = __match_any_sync(0xffffffffu, valid ? b : 0xFFFFFFFFu);
        const uint32_t wrank = __popc(peers & ((1u << lane) - 1u));
        if (valid && wrank == 0) wcnt[warp][b] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t r = running[b] + wrank;
            for (int w2 = 0; w2 < warp; ++w2) r += wcnt[w2][b];
            uint32_t k = 0;  // banks whose count is <= r (they are exhausted before round r)
#pragma unroll
            for (uint32_t step = 32; step; step >>= 1)
                if (k + step <= 32u && sorted_cnt[k + step - 1] <= r) k += step;
            place(prefix[k] + (32u - k) * r + __popc(sufmask[k] & ((1u << b) - 1u)), v);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t add = 0;
            for (int w2 = 0; w2 < 8; ++w2) add += wcnt[w2][tid];
            running[tid] += add;
        }
        __syncthreads();
    }
}

struct SlArgs {
    const uint64_t *literals;
    const uint32_t *lit_start;
    const uint64_t *tile_lbase;
    const uint4 *events;
    const uint64_t *tile_ebase;
    const uint4 *tile_desc;
    const uint32_t *tile_order;
    const TileMeta *tile_meta;
    SlicedEval e;
};

// The tile's list descriptor (see slice_scan_kernel).
struct EvDesc {
    uint4 a, b, c;  // ends: a.x..a.w, b.x, b.y; real lengths: b.z, b.w, c.x..c.w
};

// Three 10-bit events of one 32-bit word, stored as byte offsets into the difference
// array (position * 4 in bits 2-11, 12-21, 22-31: one LOP3 for the first, a shift and
// a LOP3 for the others): event j of the vector is field j mod 3 of word j / 3;
// events j with 32 j >= limit are padding.
template <int J0>
__device__ __forceinline__ void add_events(uint32_t *cnt, uint32_t w, uint32_t delta, int limit) {
#pragma unroll
    for (int f = 0; f < 3; ++f)
        if ((J0 + f) * 32 < limit)
            atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + ((w >> (10 * f)) & 0xFFCu)), delta);
}

// Row descriptor of the warp row starting at vector g of the tile: the constant of
// its list and the real events left in the list from the row's start (lists are
// padded to whole rows, so every row lies in one list).  Vector lane of the row holds
// the row's events 32 j + lane, j < 12.
__device__ __forceinline__ uint2 row_desc(uint32_t g, const EvDesc &ed) {
    uint32_t delta, start, real;
    if (g < ed.a.x) delta = 1u, start = 0u, real = ed.b.z;
    else if (g < ed.a.y) delta = 0xFFFFFFFFu, start = ed.a.x, real = ed.b.w;
    else if (g < ed.a.z) delta = 0x10000u, start = ed.a.y, real = ed.c.x;
    else if (g < ed.a.w) delta = 0xFFFF0000u, start = ed.a.z, real = ed.c.y;
    else if (g < ed.b.x) delta = 0xFFFF0001u, start = ed.a.w, real = ed.c.z;
    else delta = 0x0000FFFFu, start = ed.b.x, real = ed.c.w;
    return make_uint2(delta, real - (g - start) / 32 * kEvRow);
}

// One 16-byte vector (12 events) of a row with descriptor rd, at lane `lane`.
__device__ __forceinline__ void add_vector(uint32_t *cnt, const uint4 v, const uint2 rd, int lane) {
    const int limit = (int)rd.y - lane;
    if (limit >= kEvRow) {  // every row but a list's last: no padding
        add_events<0>(cnt, v.x, rd.x, kEvRow);
        add_events<3>(cnt, v.y, rd.x, kEvRow);
        add_events<6>(cnt, v.z, rd.x, kEvRow);
        add_events<9>(cnt, v.w, rd.x, kEvRow);
    } else {
        add_events<0>(cnt, v.x, rd.x, limit);
        add_events<3>(cnt, v.y, rd.x, limit);
        add_events<6>(cnt, v.z, rd.x, limit);
        add_events<9>(cnt, v.w, rd.x, limit);
    }
}

__device__ __forceinline__ void full_add(uint64_t a, uint64_t b, uint64_t c, uint64_t &s, uint64_t &cy) {
    s = a ^ b ^ c;                    // LOP3 0x96
    cy = (a & b) | (c & (a ^ b));     // LOP3 0xE8
}

// Bit-sliced sum (planes 0..M-1 of the 64 per-bit counts, M >= 3) of n contiguous
// literal words: full groups of 7 loaded at once and reduced by a 4-adder carry-save
// tree to a 3-bit bit-sliced number, which is then added into the planes; the last
// words rippled in one at a time.
template <int M>
__device__ __forceinline__ void planes_sum_contig(const uint64_t *p, uint32_t n, uint64_t (&c)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = 0ull;
    uint32_t i = 0;
    for (; i + 7 <= n; i += 7) {
        uint64_t x[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) x[k] = __ldg(p + i + k);
        uint64_t a0, a1, b0, b1, s1, c1, s2, s4, cy, t;
        full_add(x[0], x[1], x[2], a0, a1);
        full_add(x[3], x[4], x[5], b0, b1);
        full_add(a0, b0, x[6], s1, c1);
        full_add(a1, b1, c1, s2, s4);
        cy = c[0] & s1;
        c[0] ^= s1;
        full_add(c[1], s2, cy, t, cy);
        c[1] = t;
        full_add(c[2], s4, cy, t, cy);
        c[2] = t;
#pragma unroll
        for (int j = 3; j < M; ++j) {
            t = c[j] & cy;
            c[j] ^= cy;
            cy = t;
        }
    }
    for (; i < n; ++i) ripple<M>(c, __ldg(p + i));
}

// Write result word p of the tile (masked past r); returns its popcount.
__device__ __forceinline__ unsigned long long sl_store(const TileDecide &d, uint32_t p, uint64_t w) {
    if (d.ts + p == d.total_words - 1) w &= d.last_mask;
    d.out[d.ts - d.out_first + p] = w;
    return __popcll(w);
}

__device__ __forceinline__ void sl_finish(unsigned long long pc, int lane, unsigned long long *popcnt) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_down_sync(0xffffffffu, pc, o);
    if (lane == 0 && pc && popcnt) atomicAdd(popcnt, pc);
}

__global__ void __launch_bounds__(kSlNT, BQ_SL_MINB) rle_sliced_kernel(const __grid_constant__ SlArgs a) {
    constexpr int NT = kSlNT;
    extern __shared__ __align__(128) uint8_t sl_smem[];
    // static: its address is a constant, so every update is ATOMS [offset + imm]
    __shared__ __align__(16) uint32_t cnt[kSlCntWords];
    uint64_t *bars = reinterpret_cast<uint64_t *>(sl_smem);
    uint8_t *region = sl_smem + 16;
    uint4 *buf = reinterpret_cast<uint4 *>(region);  // [2][kPieceVecs]
    __shared__ uint32_t n_undecided, n_heavy;
    __shared__ uint2 rowtab[2][kPieceVecs / 32];  // row descriptors of the staged pieces
    __shared__ uint32_t warp_sums[NT / 32], warp_reach[NT / 32];

    const SlicedEval &E = a.e;
    uint32_t tile;  // tile of the query's range
    EvDesc ee;
    const uint4 *tev;
    if (a.tile_meta) {  // schedule order: one metadata load
        const TileMeta &tm = a.tile_meta[blockIdx.x];
        ee = EvDesc{tm.desc[0], tm.desc[1], tm.desc[2]};
        tev = a.events + tm.ebase;
        tile = tm.tile;
    } else {  // layout build (reach pass): tile order
        tile = blockIdx.x;
        ee = EvDesc{a.tile_desc[3 * tile], a.tile_desc[3 * tile + 1], a.tile_desc[3 * tile + 2]};
        tev = a.events + a.tile_ebase[tile];
    }
    const uint64_t ts = (uint64_t)(E.tile0 + tile) * kRleTile;
    const int width = (int)min((uint64_t)kRleTile, E.total_words - ts);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nvec = ee.b.y;
    const uint32_t npieces = (nvec + kPieceVecs - 1) / kPieceVecs;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);

    auto issue = [&](uint32_t p) {  // thread 0: stage piece p into buf[p & 1]
        const uint32_t nv = min((uint32_t)kPieceVecs, nvec - p * kPieceVecs);
        const uint32_t bytes = nv * 16;
        const uint32_t bar = bar0 + 8 * (p & 1);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + (size_t)(p & 1) * kPieceVecs);
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
                     "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                     "l"(tev + (size_t)p * kPieceVecs), "r"(bytes), "r"(bar)
                     : "memory");
    };

    auto fill_rows = [&](uint32_t p) {  // threads < rows per piece: descriptors of piece p's rows
        const uint32_t g = p * kPieceVecs + tid * 32;
        if (tid < kPieceVecs / 32 && g < nvec) rowtab[p & 1][tid] = row_desc(g, ee);
    };
    fill_rows(0);
    for (int k = tid; k < kSlCntWords; k += NT) cnt[k] = 0u;
    if (tid == 0) {
        n_undecided = 0;
        n_heavy = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (E.debug < 2) {
            if (npieces > 0) issue(0);
            if (npieces > 1) issue(1);
        }
    }
    __syncthreads();

    // ---- A: the tile's events into the difference array ---------------------------
    for (uint32_t p = 0; p < npieces && E.debug < 2; ++p) {
        const uint32_t bar = bar0 + 8 * (p & 1), parity = (p >> 1) & 1;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                : "=r"(done)
                : "r"(bar), "r"(parity)
                : "memory");
        }
        const uint32_t nv = min((uint32_t)kPieceVecs, nvec - p * kPieceVecs);
        const uint4 *pb = buf + (size_t)(p & 1) * kPieceVecs;
        const uint32_t g0 = p * kPieceVecs;
        if (!E.debug) {
            const uint2 *rt = rowtab[p & 1];
            uint32_t i = tid;
            for (; i + NT < nv; i += 2 * NT) {  // two vectors per iteration: both shared loads ahead of the updates
                const uint4 v0 = pb[i], v1 = pb[i + NT];
                add_vector(cnt, v0, rt[i >> 5], lane);
                add_vector(cnt, v1, rt[(i + NT) >> 5], lane);
            }
            if (i < nv) add_vector(cnt, pb[i], rt[i >> 5], lane);
        }
        fill_rows(p + 1);  // into the other table: piece p - 1's, free since the last barrier
        __syncthreads();  // buf[p & 1] is free
        if (tid == 0 && p + 2 < npieces) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(p + 2);
        }
    }
    __syncthreads();

    // ---- B: prefix sum, then decide every word the fills decide ------------------
    const uint32_t reach = tile_scan<NT>(cnt, warp_sums, warp_reach);
    if (E.reach_out) {
        if (tid == 0) E.reach_out[tile] = reach;
        return;
    }
    TileDecide d{ts, width, E.total_words, E.last_mask, E.accept_bits, E.const_until, E.out, (uint64_t)E.tile0 * kRleTile,
                 E.breaks, E.nbreak};
    uint16_t *undecided = reinterpret_cast<uint16_t *>(region);  // [kRleTile]
    uint16_t *heavy = undecided + kRleTile;                      // [kRleTile]
    unsigned long long pc = tile_decide<NT>(d, cnt, reach, undecided, &n_undecided);
    __syncthreads();
    const uint32_t nu = n_undecided;
    if (!nu) {
        sl_finish(pc, lane, E.popcnt);
        return;
    }
    const uint64_t lbase = a.tile_lbase[tile];
    const uint32_t nlit = (uint32_t)(a.tile_lbase[tile + 1] - lbase);
    const uint64_t *tlit = a.literals + lbase;
    const uint32_t *tls = a.lit_start + (size_t)tile * kLitStarts;
    if (tid == 0) {  // phase C reads the tile's literal offsets and some of its literals
        auto prefetch = [](const void *from, const void *to) {
            const uint64_t p0 = reinterpret_cast<uint64_t>(from) & ~15ull;
            const uint64_t p1 = (reinterpret_cast<uint64_t>(to) + 15) & ~15ull;
            for (uint64_t p = p0; p < p1; p += 1u << 16)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"((uint32_t)min(p1 - p, (uint64_t)1 << 16)));
        };
        prefetch(tls, tls + kRleTile);
        prefetch(tlit, tlit + nlit);
    }

    // ---- C: literal bits of undecided words ---------------------------------------
    // A word's literal words are contiguous (position-major literals): one thread
    // sums them into bit-sliced counters in registers and decides all 64 bits with
    // bit-sliced comparisons (runmerge.py:99-125's per-bit count, 64 positions at a
    // time); words with many literals go to a warp each.
    for (uint32_t u = tid; u < nu; u += NT) {
        const uint32_t p = undecided[u];
        const uint32_t c = cnt[p], ones = c & 0xFFFFu, dirty = c >> 16;
        if (dirty >= kThreadWordMax) {
            heavy[atomicAdd(&n_heavy, 1u)] = (uint16_t)p;
            continue;
        }
        const uint64_t *lits = tlit + __ldg(tls + p);
        uint64_t planes[16];
        if (dirty < 16) {
            planes_sum_contig<4>(lits, dirty, planes);
            pc += sl_store(d, p, decide_word<4>(d, ones, dirty, planes));
        } else {
            planes_sum_contig<7>(lits, dirty, planes);
            pc += sl_store(d, p, decide_word<7>(d, ones, dirty, planes));
        }
    }
    __syncthreads();
    for (uint32_t h = warp; h < n_heavy; h += NT / 32) {
        const uint32_t p = heavy[h];
        const uint32_t c = cnt[p], ones = c & 0xFFFFu, dirty = c >> 16;
        const uint64_t *lits = tlit + __ldg(tls + p);
        uint32_t c_lo = 0, c_hi = 0;  // this lane's bit positions: lane, lane + 32
        for (uint32_t j0 = 0; j0 < dirty; j0 += 32) {
            const uint64_t x = j0 + lane < dirty ? __ldg(lits + j0 + lane) : 0ull;
#pragma unroll
            for (int b = 0; b < 32; ++b) {
                const uint32_t lo = __popc(__ballot_sync(0xffffffffu, (x >> b) & 1u));
                const uint32_t hi = __popc(__ballot_sync(0xffffffffu, (x >> (b + 32)) & 1u));
                if (lane == b) {
                    c_lo += lo;
                    c_hi += hi;
                }
            }
        }
        const uint64_t w = (uint64_t)__ballot_sync(0xffffffffu, accept_at(d.accept_bits, ones + c_lo)) |
                           ((uint64_t)__ballot_sync(0xffffffffu, accept_at(d.accept_bits, ones + c_hi)) << 32);
        if (lane == 0) pc += sl_store(d, p, w);
    }
    sl_finish(pc, lane, E.popcnt);
}


}  // namespace

int build_sliced(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const uint2 *d_dir, int n, uint32_t tile0,
                 uint32_t ntiles, SlicedLayout *out) {
    *out = SlicedLayout();
    if (!ntiles) return BQ_OK;
    const uint64_t cells = (uint64_t)ntiles * n;
    const size_t T1 = (size_t)ntiles + 1;
    // scratch: slice event counts / offsets (32 B per slice) | slice marker and literal
    // counts / offsets | tile marker (statistic), literal, event totals and their scans | list ends
    // | real list lengths | CUB temp
    size_t tmp_bytes = 0, tmp2 = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                                  (int64_t)T1);
    if (e != cudaSuccess) return cuda_error(e, "DeviceScan sizing");
    const size_t scratch_bytes = cells * 40 + 6 * T1 * 8 + 16 + T1 * 48 + tmp_bytes + 256;
    char *scratch = nullptr;
    e = pool_alloc(reinterpret_cast<void **>(&scratch), scratch_bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return BQ_OK;  // no room: the query keeps the per-stream layout
    }
    ulonglong4 *ecounts = reinterpret_cast<ulonglong4 *>(scratch);
    uint64_t *counts = reinterpret_cast<uint64_t *>(ecounts + cells);
    uint64_t *tm = counts + cells, *tl = tm + T1, *te = tl + T1, *mb = te + T1, *lb = mb + T1, *eb = lb + T1;
    uint4 *desc = reinterpret_cast<uint4 *>(scratch + ((reinterpret_cast<char *>(eb + T1) - scratch) + 15) / 16 * 16);
    void *d_tmp = desc + 3 * T1;
    const int sms = sm_count();
    const unsigned grid = (unsigned)std::min<uint64_t>((cells + 255) / 256, (uint64_t)sms * 32);
    char *evsrc = nullptr;
    auto fail = [&](cudaError_t err, const char *what) {
        pool_free(scratch);
        if (evsrc) pool_free(evsrc);
        return cuda_error(err, what);
    };
    slice_count_kernel<<<grid, 256>>>(d_ptrs, d_lens, d_dir, n, tile0, ntiles, counts, ecounts);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemset(tm + ntiles, 0, 8);
    if (e == cudaSuccess) e = cudaMemset(tl + ntiles, 0, 8);
    if (e == cudaSuccess) e = cudaMemset(te + ntiles, 0, 8);
    if (e != cudaSuccess) return fail(e, "slice_count_kernel");
    slice_scan_kernel<<<ntiles, 1024>>>(counts, ecounts, n, tm, tl, te, desc);
    e = cudaGetLastError();
    tmp2 = tmp_bytes;
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp2, tm, mb, (int64_t)T1);
    tmp2 = tmp_bytes;
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp2, tl, lb, (int64_t)T1);
    tmp2 = tmp_bytes;
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp2, te, eb, (int64_t)T1);
    uint64_t nm = 0, nl = 0, ne = 0;  // ne: event vectors
    if (e == cudaSuccess) e = cudaMemcpy(&nm, mb + ntiles, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&nl, lb + ntiles, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&ne, eb + ntiles, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(e, "slice scans");
    // literals | tile_lbase | lit_start | events | tile_ebase | tile_desc | tile_order
    // (literals, events and tile_desc at 16-byte boundaries)
    auto r16 = [](size_t x) { return (x + 15) / 16 * 16; };
    const size_t o_tlb = nl * 8;
    const size_t o_ls = o_tlb + T1 * 8;
    const size_t o_ev = r16(o_ls + (size_t)ntiles * kLitStarts * 4);
    const size_t o_teb = o_ev + ne * 16;
    const size_t o_tee = r16(o_teb + T1 * 8);
    const size_t o_ord = o_tee + (size_t)ntiles * 48;
    const size_t o_meta = (o_ord + (size_t)ntiles * 4 + 63) / 64 * 64;
    const size_t bytes = o_meta + (size_t)ntiles * sizeof(TileMeta);
    char *m = nullptr, *tmpl = nullptr;  // tmpl: literals and positions as emitted, slice by slice
    e = pool_alloc(reinterpret_cast<void **>(&m), bytes);
    if (e == cudaSuccess && ne) e = pool_alloc(reinterpret_cast<void **>(&evsrc), ne * kEvVec * 2);  // event positions as emitted, slice by slice
    if (e == cudaSuccess) e = pool_alloc(reinterpret_cast<void **>(&tmpl), nl * 10 + 16);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (m) pool_free(m);
        if (evsrc) pool_free(evsrc);
        pool_free(scratch);
        return BQ_OK;
    }
    SlicedLayout l;
    l.mem = m;
    uint64_t *literals = reinterpret_cast<uint64_t *>(m);
    uint64_t *tlb = reinterpret_cast<uint64_t *>(m + o_tlb);
    uint32_t *lit_start = reinterpret_cast<uint32_t *>(m + o_ls);
    uint4 *events = reinterpret_cast<uint4 *>(m + o_ev);
    uint64_t *teb = reinterpret_cast<uint64_t *>(m + o_teb);
    uint4 *tee = reinterpret_cast<uint4 *>(m + o_tee);
    uint64_t *lit_src = reinterpret_cast<uint64_t *>(tmpl);
    uint16_t *pos_src = reinterpret_cast<uint16_t *>(tmpl + nl * 8);
    e = cudaMemcpy(tlb, lb, T1 * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(teb, eb, T1 * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(tee, desc, (size_t)ntiles * 48, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemset(events, 0, ne * 16);  // packed by atomicOr
    if (e == cudaSuccess) {
        slice_emit_kernel<<<grid, 256>>>(d_ptrs, d_lens, d_dir, n, tile0, ntiles, counts, ecounts, tlb, teb, tee,
                                         lit_src, pos_src, reinterpret_cast<uint16_t *>(evsrc));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        sort_literals_kernel<<<ntiles, 512>>>(lit_src, pos_src, tlb, literals, lit_start);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && ne) {
        arrange_events_kernel<<<dim3(ntiles, kEvKinds), 256>>>(reinterpret_cast<const uint16_t *>(evsrc),
                                                              reinterpret_cast<uint32_t *>(events), teb, tee);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    pool_free(scratch);
    pool_free(tmpl);
    if (evsrc) pool_free(evsrc);
    if (e != cudaSuccess) {
        pool_free(m);
        return cuda_error(e, "slice_emit_kernel / sort_literals_kernel / arrange_events_kernel");
    }
    // tile order: a reach-only pass of K4s, then tiles sorted by descending reach
    uint32_t *order = reinterpret_cast<uint32_t *>(m + o_ord);
    {
        char *ss = nullptr;
        size_t sort_bytes = 0;
        e = cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                      (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)ntiles);
        if (e == cudaSuccess) e = pool_alloc(reinterpret_cast<void **>(&ss), (size_t)ntiles * 12 + 16 + sort_bytes);
        if (e != cudaSuccess) {
            pool_free(m);
            return cuda_error(e, "tile order scratch");
        }
        uint32_t *reach = reinterpret_cast<uint32_t *>(ss), *reach_sorted = reach + ntiles, *ids = reach_sorted + ntiles;
        void *sort_tmp = ss + ((size_t)ntiles * 12 + 15) / 16 * 16;
        SlicedLayout tmp;
        tmp.literals = literals;
        tmp.lit_start = lit_start;
        tmp.tile_lbase = tlb;
        tmp.events = events;
        tmp.tile_ebase = teb;
        tmp.tile_desc = tee;
        SlicedEval re{};
        re.n = n;
        re.total_words = ~0ull;
        re.tile0 = tile0;
        re.ntiles = ntiles;
        re.reach_out = reach;
        int rc = launch_sliced(tmp, re, 0);
        if (rc) {
            pool_free(ss);
            pool_free(m);
            return rc;
        }
        iota_kernel<<<(ntiles + 255) / 256, 256>>>(ids, ntiles);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairsDescending(sort_tmp, sort_bytes, reach, reach_sorted, ids, order, (int)ntiles);
        if (e == cudaSuccess) {
            gather_meta_kernel<<<(ntiles + 255) / 256, 256>>>(order, tee, teb, reinterpret_cast<TileMeta *>(m + o_meta),
                                                             ntiles);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        pool_free(ss);
        if (e != cudaSuccess) {
            pool_free(m);
            return cuda_error(e, "tile order");
        }
    }
    l.tile_order = order;
    l.tile_meta = reinterpret_cast<const TileMeta *>(m + o_meta);
    l.literals = literals;
    l.lit_start = lit_start;
    l.tile_lbase = tlb;
    l.events = events;
    l.tile_ebase = teb;
    l.tile_desc = tee;
    l.bytes = bytes;
    l.n_markers = nm;
    l.n_literals = nl;
    l.n_events = ne * kEvVec;
    *out = l;
    return BQ_OK;
}

void free_sliced(SlicedLayout *l, const StreamUses *uses) {
    if (l->mem) {
        if (uses)
            pool_free_after(l->mem, *uses);
        else
            pool_free(l->mem);
    }
    *l = SlicedLayout();
}

int launch_sliced(const SlicedLayout &l, const SlicedEval &e, cudaStream_t stream) {
    SlArgs a;
    a.literals = l.literals;
    a.lit_start = l.lit_start;
    a.tile_lbase = l.tile_lbase;
    a.events = l.events;
    a.tile_ebase = l.tile_ebase;
    a.tile_desc = l.tile_desc;
    a.tile_order = e.reach_out ? nullptr : l.tile_order;
    a.tile_meta = e.reach_out ? nullptr : l.tile_meta;
    a.e = e;
    cudaError_t err = cudaFuncSetAttribute(rle_sliced_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlSmem);
    if (err != cudaSuccess) return cuda_error(err, "cudaFuncSetAttribute(rle_sliced_kernel)");
    rle_sliced_kernel<<<e.ntiles, kSlNT, kSlSmem, stream>>>(a);
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_error(err, "rle_sliced_kernel launch");
    return BQ_OK;
}

}  // namespace bq
