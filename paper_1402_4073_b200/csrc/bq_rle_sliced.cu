// K4 over the tile-sliced RLE layout (see SlicedLayout in bq_internal.h).
//
// The per-stream K4 (bq_rle.cu) gives each lane one stream and follows its
// marker chain: a dependent shared-memory load per marker, and lanes idle while
// the longest chain of the warp finishes (~47% lane efficiency on C4).  Here the
// streams are re-encoded once per query into 1024-word slices whose markers are
// contiguous per tile and cover exactly 1024 words each, so the word position of
// a marker is the running sum of (run + dirty) modulo 1024 -- a warp prefix sum
// over 128 markers at a time (4 per lane) replaces the chain walk, every lane is
// busy, and phase A reads only the 32-bit markers (literal words are read in
// phase C, only at undecided positions, as runmerge.cdom_threshold examines
// dirty words only where the fill counts do not decide; runmerge.py:198-241).
//
// Per tile (one CTA): A) markers staged into shared memory by TMA bulk copies in
// 16 KB pieces (double-buffered); each chunk of 128 markers is decoded by one
// warp into the packed difference array cnt (ones | dirty << 16); B) prefix sum
// and const_until decisions; C) bit counters of undecided words from their
// literals.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "bq_internal.h"
#include "bq_rle_tile.cuh"

namespace bq {

namespace {

#ifndef BQ_SL_NT
#define BQ_SL_NT 128
#define BQ_SL_MINB 5
#endif
#ifndef BQ_SL_SLOTS
#define BQ_SL_SLOTS 256
#endif
constexpr int kSlNT = BQ_SL_NT;                            // K4s threads per CTA (4 warps)
constexpr int kPieceChunks = 32;                           // chunks per staged piece
constexpr int kPieceMarkers = kPieceChunks * kSliceChunk;  // 4096 markers = 16 KB
constexpr int kSlSlots = BQ_SL_SLOTS;                      // undecided words per phase-C pass
constexpr size_t kSlCntBytes = (size_t)(kRleTile + 36) * 4;  // + sentinel + 32 per-lane dummies (+ pad)
constexpr size_t kSlBufBytes = 2 * (size_t)kPieceMarkers * 4;
constexpr size_t kSlPhaseC = tile_resolve_bytes<kSlSlots>() + (size_t)kRleTile * 2;  // + undecided list
constexpr size_t kSlRegion = kSlBufBytes > kSlPhaseC ? kSlBufBytes : kSlPhaseC;
constexpr size_t kSlSmem = kSlCntBytes + 16 + kSlRegion;  // cnt | 2 mbarriers | region

// 32-bit slice marker: run (bits 0-10) | fill bit (bit 11) | dirty (bits 16-26); run, dirty <= 1024
__device__ __forceinline__ uint32_t mk_bit(uint32_t m) { return (m >> 11) & 1u; }
__device__ __forceinline__ uint32_t mk_run(uint32_t m) { return m & 0x7FFu; }
__device__ __forceinline__ uint32_t mk_dirty(uint32_t m) { return m >> 16; }
__device__ __forceinline__ uint32_t mk_pack(uint32_t bit, uint32_t run, uint32_t dirty) { return run | (bit << 11) | (dirty << 16); }

// ---------------------------------------------------------------------------
// Layout build, one thread per (tile, stream) slice.  The counting pass maps
// neighbouring threads to neighbouring tiles of one stream (their reads are
// adjacent); the emitting pass to neighbouring streams of one tile (their writes
// are adjacent in the tile-major output): 0.9 + 3.0 ms at C4 instead of 0.9 + 5.3.

struct SliceSink {
    uint32_t *mk;       // tile marker array (null: count only)
    uint64_t *lit;      // tile literal array
    uint64_t *meta;     // chunk checkpoints of this tile
    uint32_t mk0, lit0;  // within-tile index of the slice's first marker / literal
};

// Re-encode stream words [ts, ts + 1024) starting at the directory entry e
// (marker index, fill start).  Returns (markers, literals) of the slice.
template <bool EMIT>
__device__ uint2 slice_walk(const uint64_t *src, uint64_t L, uint2 e, uint64_t ts, const SliceSink &sink) {
    const uint64_t te = ts + kRleTile;
    uint64_t i = e.x, pos = e.y;
    uint32_t rel = 0, n_mk = 0, n_lit = 0;
    bool prev_dirty = false;
    auto emit = [&](uint32_t bit, uint32_t run, uint32_t dirty) {
        if (EMIT) {
            const uint32_t j = sink.mk0 + n_mk;
            sink.mk[j] = mk_pack(bit, run, dirty);
            if (j % kSliceChunk == 0)
                sink.meta[j / kSliceChunk] = (uint64_t)rel | ((uint64_t)(rel != 0 && prev_dirty) << 11) |
                                             ((uint64_t)(sink.lit0 + n_lit) << 32);
        }
        ++n_mk;
        rel += run + dirty;
        prev_dirty = dirty != 0;
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
                for (uint32_t k = 0; k < cdirty; ++k) sink.lit[sink.lit0 + n_lit + k] = __ldg(src + i + 1 + (cds - fe) + k);
            emit((uint32_t)(m & 1) & (crun != 0u), crun, cdirty);
            n_lit += cdirty;
        }
        pos = de;
        i += 1 + dirty;
    }
    return make_uint2(n_mk, n_lit);
}

__global__ void slice_count_kernel(const uint64_t *const *ptrs, const uint64_t *lens, const uint2 *dir, int n,
                                   uint32_t tile0, uint32_t ntiles, uint64_t *counts) {
    const uint64_t total = (uint64_t)ntiles * n;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const int s = (int)(k / ntiles);  // neighbouring threads: neighbouring tiles of one stream (reads)
        const uint32_t t = (uint32_t)(k % ntiles);
        const uint2 c =
            slice_walk<false>(ptrs[s], lens[s], dir[(size_t)t * n + s], (uint64_t)(tile0 + t) * kRleTile, SliceSink{});
        counts[(size_t)t * n + s] = (uint64_t)c.x | ((uint64_t)c.y << 32);
    }
}

// One CTA per tile: exclusive scan of the slice counts in place (markers in the low,
// literals in the high half: each half of a tile's sum stays below 2^32), and the
// tile totals, markers rounded up to whole chunks.
__global__ void __launch_bounds__(1024) slice_scan_kernel(uint64_t *counts, int n, uint64_t *tile_m, uint64_t *tile_l) {
    using Scan = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint64_t carry;
    const uint32_t t = blockIdx.x;
    uint64_t *row = counts + (size_t)t * n;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int s = base + (int)threadIdx.x;
        const uint64_t v = s < n ? row[s] : 0ull;
        uint64_t ex, agg;
        Scan(tmp).ExclusiveSum(v, ex, agg);
        const uint64_t c = carry;
        if (s < n) row[s] = ex + c;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint64_t m = carry & 0xFFFFFFFFull, l = carry >> 32;
        tile_m[t] = (m + kSliceChunk - 1) / kSliceChunk * kSliceChunk;
        tile_l[t] = l;
    }
}

__global__ void slice_emit_kernel(const uint64_t *const *ptrs, const uint64_t *lens, const uint2 *dir, int n,
                                  uint32_t tile0, uint32_t ntiles, const uint64_t *offs, const uint64_t *mbase, const uint64_t *lbase,
                                  uint32_t *markers, uint64_t *literals, uint64_t *meta) {
    const uint64_t total = (uint64_t)ntiles * n;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const int s = (int)(k % n);  // neighbouring threads: neighbouring slices of one tile (writes)
        const uint32_t t = (uint32_t)(k / n);
        const uint64_t o = offs[(size_t)t * n + s];
        SliceSink sink;
        sink.mk = markers + mbase[t];
        sink.lit = literals + lbase[t];
        sink.meta = meta + mbase[t] / kSliceChunk;
        sink.mk0 = (uint32_t)o;
        sink.lit0 = (uint32_t)(o >> 32);
        slice_walk<true>(ptrs[s], lens[s], dir[(size_t)t * n + s], (uint64_t)(tile0 + t) * kRleTile, sink);
    }
}

// ---------------------------------------------------------------------------
// K4s: one CTA per tile.

// K4s decode is bound by the ALU pipe (shifts, masks, selects, LEA); the shared-memory
// byte offsets are formed as index * four with four a runtime value, so they go to
// the FMA pipe (IMAD) instead of an ALU LEA.
struct MulC {
    uint32_t four;  // 4
};

struct SlArgs {
    const uint32_t *markers;
    const uint64_t *literals;
    const uint64_t *tile_mbase, *tile_lbase, *chunk_meta;
    MulC mc;
    SlicedEval e;
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) { return warp_incl_scan_u32(v, lane); }

// Decode one chunk (4 markers per lane) into the difference array: the word
// position of each marker is the chunk checkpoint plus the warp prefix sum of
// (run + dirty), modulo 1024 (slices cover exactly 1024 words).  Two updates per
// marker: (+one-fill start, -pending literal end) at its start, (-one-fill end,
// +literal start) where its fill ends.

__device__ __forceinline__ void decode_chunk(const uint4 v, uint32_t cm, int lane, uint32_t *cnt, const MulC &c) {
    const uint32_t four = c.four;
    const uint32_t dummy = kRleTile + 1 + lane;  // per-lane slot for zero updates (no same-address conflicts)
    const uint32_t m[4] = {v.x, v.y, v.z, v.w};
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) tot += mk_run(m[k]) + mk_dirty(m[k]);
    const uint32_t incl = warp_incl_scan(tot, lane);
    uint32_t rel = (cm + incl - tot) & (kRleTile - 1);
    const uint32_t up = __shfl_up_sync(0xffffffffu, mk_dirty(m[3]), 1);
    bool pd = lane ? (up != 0u) : ((cm >> 11) & 1u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t bit = mk_bit(m[k]), run = mk_run(m[k]), dirty = mk_dirty(m[k]);
        const uint32_t fe = rel + run;
        const uint32_t at_rel = bit + ((rel != 0u && pd) ? 0xFFFF0000u : 0u);
        const uint32_t at_fe = (dirty ? 0x10000u : 0u) - bit;
        // byte offsets through IMAD (runtime stride): keeps address arithmetic off the ALU pipe
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + (at_rel ? rel : dummy) * four), at_rel);
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + (at_fe ? fe : dummy) * four), at_fe);
        pd = dirty != 0u;
        rel = (fe + dirty) & (kRleTile - 1);
    }
}

__global__ void __launch_bounds__(kSlNT, BQ_SL_MINB) rle_sliced_kernel(const __grid_constant__ SlArgs a) {
    constexpr int NT = kSlNT;
    extern __shared__ __align__(128) uint8_t sl_smem[];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(sl_smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sl_smem + kSlCntBytes);
    uint8_t *region = sl_smem + kSlCntBytes + 16;
    uint32_t *buf = reinterpret_cast<uint32_t *>(region);  // [2][kPieceMarkers]
    __shared__ uint32_t n_undecided;
    __shared__ uint32_t warp_sums[NT / 32], warp_reach[NT / 32];

    const SlicedEval &E = a.e;
    const uint32_t tile = blockIdx.x;  // tile of the query's range; its words are global
    const uint64_t ts = (uint64_t)(E.tile0 + tile) * kRleTile;
    const int width = (int)min((uint64_t)kRleTile, E.total_words - ts);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t mbase = a.tile_mbase[tile];
    const uint32_t nchunks = (uint32_t)((a.tile_mbase[tile + 1] - mbase) / kSliceChunk);
    const uint64_t *meta = a.chunk_meta + mbase / kSliceChunk;
    const uint32_t *tmk = a.markers + mbase;
    const uint64_t *tlit = a.literals + a.tile_lbase[tile];
    const uint32_t npieces = (nchunks + kPieceChunks - 1) / kPieceChunks;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);

    auto issue = [&](uint32_t p) {  // thread 0: stage piece p into buf[p & 1]
        const uint32_t nc = min((uint32_t)kPieceChunks, nchunks - p * kPieceChunks);
        const uint32_t bytes = nc * kSliceChunk * 4;
        const uint32_t bar = bar0 + 8 * (p & 1);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + (size_t)(p & 1) * kPieceMarkers);
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
                     "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                     "l"(tmk + (size_t)p * kPieceMarkers), "r"(bytes), "r"(bar)
                     : "memory");
    };

    for (int k = tid; k < kRleTile + 36; k += NT) cnt[k] = 0u;
    if (tid == 0) {
        n_undecided = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (E.debug < 2) {
            if (npieces > 0) issue(0);
            if (npieces > 1) issue(1);
        }
    }
    __syncthreads();

    // ---- A: decode chunks into the difference array ----------------------------
    // chunk checkpoints of a piece, one per lane (kPieceChunks == 32), loaded a piece ahead
    auto piece_meta = [&](uint32_t p) {
        return (p < npieces && p * kPieceChunks + lane < nchunks) ? __ldg(meta + p * kPieceChunks + lane) : 0ull;
    };
    uint64_t next_meta = piece_meta(0);
    for (uint32_t p = 0; p < npieces && E.debug < 2; ++p) {
        const uint64_t pmeta = next_meta;
        next_meta = piece_meta(p + 1);
        const uint32_t bar = bar0 + 8 * (p & 1), parity = (p >> 1) & 1;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                : "=r"(done)
                : "r"(bar), "r"(parity)
                : "memory");
        }
        const uint32_t nc = min((uint32_t)kPieceChunks, nchunks - p * kPieceChunks);
        const uint4 *pb = reinterpret_cast<const uint4 *>(buf + (size_t)(p & 1) * kPieceMarkers);
        // two chunks per iteration: independent scans interleave (shuffle latency)
        for (uint32_t c = warp; c < nc && !E.debug; c += 2 * (NT / 32)) {
            const uint32_t c2 = c + NT / 32;
            const bool two = c2 < nc;
            const uint32_t cm0 = (uint32_t)__shfl_sync(0xffffffffu, pmeta, c);
            const uint32_t cm1 = (uint32_t)__shfl_sync(0xffffffffu, pmeta, two ? c2 : c);
            const uint4 v0 = pb[c * 32 + lane];
            const uint4 v1 = two ? pb[c2 * 32 + lane] : make_uint4(0u, 0u, 0u, 0u);
            decode_chunk(v0, cm0, lane, cnt, a.mc);
            decode_chunk(v1, two ? cm1 : 0u, lane, cnt, a.mc);
        }
        __syncthreads();  // buf[p & 1] is free
        if (tid == 0 && p + 2 < npieces) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(p + 2);
        }
    }
    __syncthreads();

    // ---- B: prefix sum, then decide every word the fills decide ------------------
    const uint32_t reach = tile_scan<NT>(cnt, warp_sums, warp_reach);
    TileDecide d{ts, width, E.total_words, E.last_mask, E.accept_bits, E.const_until, E.out, (uint64_t)E.tile0 * kRleTile,
                 E.breaks, E.nbreak};
    uint16_t *undecided = reinterpret_cast<uint16_t *>(region + tile_resolve_bytes<kSlSlots>());
    unsigned long long pc = tile_decide<NT>(d, cnt, reach, undecided, &n_undecided);
    __syncthreads();

    // ---- C: literal bits of undecided words (chunks decoded again, literals from HBM) --
    pc += tile_resolve<NT, kSlSlots>(d, cnt, undecided, n_undecided, region, [&](const uint16_t *slot_of,
                                                                                 auto &&add_bits) {
        for (uint32_t c = warp; c < nchunks; c += NT / 32) {
            const uint64_t cm = __ldg(meta + c);
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(tmk) + c * 32 + lane);
            const uint32_t m[4] = {v.x, v.y, v.z, v.w};
            uint32_t tot = 0, dtot = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                tot += mk_run(m[k]) + mk_dirty(m[k]);
                dtot += mk_dirty(m[k]);
            }
            const uint32_t incl_len = warp_incl_scan(tot, lane);
            const uint32_t incl_lit = warp_incl_scan(dtot, lane);
            uint32_t rel = ((uint32_t)cm + incl_len - tot) & (kRleTile - 1);
            uint32_t lit = (uint32_t)(cm >> 32) + incl_lit - dtot;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t run = mk_run(m[k]), dirty = mk_dirty(m[k]);
                const uint32_t fe = rel + run;
                for (uint32_t q = 0; q < dirty; ++q) {
                    const uint16_t u = slot_of[fe + q];
                    if (u != kNoSlot) add_bits(u, tlit + lit + q);
                }
                lit += dirty;
                rel = (fe + dirty) & (kRleTile - 1);
            }
        }
    });

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_down_sync(0xffffffffu, pc, o);
    if (lane == 0 && pc && E.popcnt) atomicAdd(E.popcnt, pc);
}

}  // namespace

int build_sliced(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const uint2 *d_dir, int n, uint32_t tile0,
                 uint32_t ntiles, SlicedLayout *out) {
    *out = SlicedLayout();
    if (!ntiles) return BQ_OK;
    const uint64_t cells = (uint64_t)ntiles * n;
    // scratch: slice counts / offsets | tile marker totals | tile literal totals | CUB temp
    size_t tmp_bytes = 0, tmp2 = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                                  (int64_t)ntiles + 1);
    if (e != cudaSuccess) return cuda_error(e, "DeviceScan sizing");
    tmp2 = tmp_bytes;
    const size_t scratch_bytes = cells * 8 + 4 * ((size_t)ntiles + 1) * 8 + tmp2 + 256;
    char *scratch = nullptr;
    e = cudaMalloc(&scratch, scratch_bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return BQ_OK;  // no room: the query keeps the per-stream layout
    }
    uint64_t *counts = reinterpret_cast<uint64_t *>(scratch);
    uint64_t *tm = counts + cells, *tl = tm + ntiles + 1, *mb = tl + ntiles + 1, *lb = mb + ntiles + 1;
    void *d_tmp = lb + ntiles + 1;
    const int sms = sm_count();
    const unsigned grid = (unsigned)std::min<uint64_t>((cells + 255) / 256, (uint64_t)sms * 32);
    auto fail = [&](cudaError_t err, const char *what) {
        cudaFree(scratch);
        return cuda_error(err, what);
    };
    slice_count_kernel<<<grid, 256>>>(d_ptrs, d_lens, d_dir, n, tile0, ntiles, counts);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemset(tm + ntiles, 0, 8);
    if (e == cudaSuccess) e = cudaMemset(tl + ntiles, 0, 8);
    if (e != cudaSuccess) return fail(e, "slice_count_kernel");
    slice_scan_kernel<<<ntiles, 1024>>>(counts, n, tm, tl);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp2, tm, mb, (int64_t)ntiles + 1);
    tmp2 = tmp_bytes;
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp2, tl, lb, (int64_t)ntiles + 1);
    uint64_t nm = 0, nl = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&nm, mb + ntiles, 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&nl, lb + ntiles, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(e, "slice scans");
    // markers (16-byte multiple) | literals | tile_mbase | tile_lbase | chunk_meta
    const size_t mk_bytes = (nm * 4 + 15) / 16 * 16;
    const size_t bytes = mk_bytes + nl * 8 + 2 * ((size_t)ntiles + 1) * 8 + nm / kSliceChunk * 8 + 64;
    char *m = nullptr;
    e = cudaMalloc(&m, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(scratch);
        return BQ_OK;
    }
    SlicedLayout l;
    l.mem = m;
    uint32_t *markers = reinterpret_cast<uint32_t *>(m);
    uint64_t *literals = reinterpret_cast<uint64_t *>(m + mk_bytes);
    uint64_t *tmb = literals + nl, *tlb = tmb + ntiles + 1, *meta = tlb + ntiles + 1;
    e = cudaMemset(markers, 0, mk_bytes);  // chunk padding decodes to empty markers
    if (e == cudaSuccess) e = cudaMemcpy(tmb, mb, ((size_t)ntiles + 1) * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(tlb, lb, ((size_t)ntiles + 1) * 8, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) {
        slice_emit_kernel<<<grid, 256>>>(d_ptrs, d_lens, d_dir, n, tile0, ntiles, counts, tmb, tlb, markers, literals,
                                         meta);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(scratch);
    if (e != cudaSuccess) {
        cudaFree(m);
        return cuda_error(e, "slice_emit_kernel");
    }
    l.markers = markers;
    l.literals = literals;
    l.tile_mbase = tmb;
    l.tile_lbase = tlb;
    l.chunk_meta = meta;
    l.bytes = bytes;
    l.n_markers = nm;
    l.n_literals = nl;
    *out = l;
    return BQ_OK;
}

void free_sliced(SlicedLayout *l) {
    if (l->mem) cudaFree(l->mem);
    *l = SlicedLayout();
}

int launch_sliced(const SlicedLayout &l, const SlicedEval &e, cudaStream_t stream) {
    SlArgs a;
    a.markers = l.markers;
    a.literals = l.literals;
    a.tile_mbase = l.tile_mbase;
    a.tile_lbase = l.tile_lbase;
    a.chunk_meta = l.chunk_meta;
    a.mc = MulC{4u};
    a.e = e;
    cudaError_t err = cudaFuncSetAttribute(rle_sliced_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlSmem);
    if (err != cudaSuccess) return cuda_error(err, "cudaFuncSetAttribute(rle_sliced_kernel)");
    rle_sliced_kernel<<<e.ntiles, kSlNT, kSlSmem, stream>>>(a);
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_error(err, "rle_sliced_kernel launch");
    return BQ_OK;
}

}  // namespace bq
