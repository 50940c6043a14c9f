// K3/K4: threshold and symmetric queries over EWAH-style run-length-encoded
// bitmaps, decoded on the device (sm_100a).
//
// Stream format (reference bitmaps.py:27-40): a marker word
//   bit 0 = fill bit, bits 1-32 = fill run (words), bits 33-63 = literal count
// followed by that many literal ("dirty") words; coverage shorter than
// ceil(r/64) words is an implicit zero tail (bitmaps.py:215-219).
//
// K3 the tile directory, once per query object (inputs are immutable): the marker
//   covering every tile boundary, found in one streaming pass with speculative
//   per-segment walks and a decoupled look-back across blocks (bq_rle_dir.cu),
//   which also validates the streams as RleBitmap.iter_word_segments (:210-217).
//
// K4 rle_count_kernel -- a query's first evaluation: the per-tile form of cdom's run
//   sweep (runmerge.py:198-299) over tiles of kRleTile output words, kWT tiles per CTA:
//   A. each lane walks one (stream, tile) slice from its directory entry, reading
//      only marker words (staged by TMA, one bulk copy per stream and kWT tiles);
//      one-fill and dirty runs become +1/-1 entries of the tile's packed
//      shared-memory difference array (ones in bits 0-15, dirty in 16-31), so a
//      prefix scan yields k_w (one-fills) and d_w (dirty inputs) for every word w;
//   B. w is decided from (k_w, d_w) alone when accept[] is constant on
//      [k_w, k_w + d_w] (cdom's three cases) -- the common
//      case -- and written directly;
//   C. only for undecided words are the dirty literals read (K4c rle_resolve_kernel,
//      over the tiles K4 lists): a second walk files their addresses, bit-sliced
//      sums count each bit position, then accept[k_w + count_b] decides each bit
//      (dirty_segment_solver's "scan" branch, runmerge.py:99-125).
//   Output is uncompressed (BASELINE config 4), with a fused popcount.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "bq_internal.h"
#include "bq_rle_tile.cuh"

namespace bq {

#ifndef BQ_K4_C_ILP
#define BQ_K4_C_ILP 4  // streams walked at once per thread in phase C
#endif

enum { RLE_ERR_TRUNCATED = 1, RLE_ERR_OVERLONG = 2, RLE_ERR_BEYOND_R = 3 };  // build_rle_directory's codes

struct RleCountArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    const uint2 *dir;
    int n;
    uint64_t total_words;
    uint32_t tile0;   // first (global) tile of the query's range; blockIdx.x is the tile within it
    uint64_t last_mask;
    const uint32_t *accept_bits;  // (n + 1) bits
    const uint32_t *const_until;  // [n + 1]: largest j >= k with accept[k..j] constant
    const uint32_t *breaks;       // counts where accept[] changes (phase C's bit-sliced decisions)
    int nbreak;                   // their number, -1 when there are too many
    uint64_t *out;
    unsigned long long *popcnt;
    int debug;  // experiment knob (BQ_RLE_DEBUG): 1 = skip marker walks, 2 = also skip copies
    uint32_t four;  // 4 as a runtime value (see sweep_stream)
    // phase C deferred to rle_resolve_kernel: a tile with undecided words appends itself to
    // todo[] and leaves its scanned counts in todo_cnt[slot][kRleTile]
    uint32_t *todo_count;
    uint32_t *todo;
    uint32_t *todo_cnt;
    uint32_t tile_off;  // K4 launches cover directory rows [tile_off, tile_off + tile_cnt)
    uint32_t tile_cnt;
};


// Walk every stream st = first, first + stride, ... < n across tile [ts, te) from its
// directory entry; visit(fs, fe, bit, ds, de, lit, s) is called for each marker whose runs
// intersect the tile (fill [fs, fe), dirty [ds, de), first literal at s[lit]).  U streams
// are walked at a time with their marker loads interleaved (U independent loads in flight
// per thread instead of one dependent chain).  A stream st < nstaged whose slice the CTA
// staged reads it from shared memory (stage_off[st] = pool word of its directory marker,
// kNotStaged otherwise; stage_end[st] = the first stream word past the staged slice: the
// literal words of the slice's last marker can extend beyond it, and those are read from
// HBM); the other streams walk HBM, latency-bound.
constexpr uint32_t kNotStaged = 0xFFFFFFFFu;
template <int U, typename Visit>
__device__ __forceinline__ void walk_tiles(const RleCountArgs &a, int first, int stride, uint32_t tile, uint64_t ts,
                                           uint64_t te, const uint64_t *pool, const uint32_t *stage_off,
                                           const uint32_t *stage_end, int nstaged, Visit &&visit) {
    for (int base = first; base < a.n; base += U * stride) {
        const uint64_t *sp[U];
        uint64_t L[U], i[U], pos[U];
        uint32_t send[U];  // staged streams: first stream word not in the pool
        bool act[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int st = base + u * stride;
            act[u] = st < a.n;
            sp[u] = nullptr;
            L[u] = i[u] = pos[u] = 0;
            send[u] = kNotStaged;
            if (act[u]) {
                sp[u] = a.ptrs[st];
                L[u] = a.lens[st];
                const uint2 e = a.dir[(size_t)tile * a.n + st];
                i[u] = e.x;
                pos[u] = e.y;
                act[u] = i[u] < L[u] && pos[u] < te;
                if (st < nstaged) {
                    const uint32_t so = stage_off[st];
                    if (so != kNotStaged) {
                        sp[u] = pool + so - e.x;  // sp[u][i] is stream word i, for e.x <= i < send[u]
                        send[u] = stage_end[st];
                    }
                }
            }
        }
        for (;;) {
            bool any = false;
#pragma unroll
            for (int u = 0; u < U; ++u) any |= act[u];
            if (!any) break;
            uint64_t mk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) mk[u] = act[u] ? sp[u][i[u]] : 0ull;  // generic: HBM or the pool
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                const uint64_t run = (mk[u] >> 1) & 0xFFFFFFFFull;
                const uint64_t dirty = mk[u] >> 33;
                const uint64_t fe = pos[u] + run, de = fe + dirty;
                if (de > ts) {
                    // literal words of this marker the tile needs: stream words [i + 1, i + 1 + (min(de, te) - fe))
                    const uint64_t need = i[u] + 1 + (min(de, te) - min(fe, te));
                    if (need <= send[u]) {
                        visit(pos[u], fe, (uint32_t)(mk[u] & 1), fe, de, i[u] + 1, sp[u]);
                    } else {  // rare: the slice's last marker, its literals run past the staged words
                        const uint64_t in_pool = send[u] > i[u] + 1 ? send[u] - (i[u] + 1) : 0;  // literals staged
                        const uint64_t cut = min(fe + in_pool, de);
                        if (cut > fe) visit(pos[u], fe, (uint32_t)(mk[u] & 1), fe, cut, i[u] + 1, sp[u]);
                        const uint64_t *gp = a.ptrs[base + u * stride];
                        visit(pos[u], fe, (uint32_t)(mk[u] & 1), cut, de, i[u] + 1 + (cut - fe), gp);
                    }
                }
                pos[u] = de;
                i[u] += 1 + dirty;
                act[u] = i[u] < L[u] && pos[u] < te;
            }
        }
    }
}


// Marker sweep of one stream over a tile of W words in 32-bit tile-relative
// coordinates.  src[0] is the marker named by the stream's directory entry
// (its fill run starts at word `pos`, at or before the tile); lim = stream
// words available from there.  Each marker adds at most three entries to the
// packed difference array: +1 at a one-fill's start, (-1 | +dirty) where the
// fill ends and the literals begin, -dirty where the literals end.
template <bool GLOBAL>
__device__ __forceinline__ void sweep_stream(const uint64_t *src, uint32_t lim, uint32_t pos, uint64_t ts, int W,
                                             uint32_t *cnt, uint32_t four, uint32_t dummy) {
    // dummy: this lane's slot (> W) for the first marker's empty contributions
    auto load = [src](uint32_t k) { return GLOBAL ? __ldg(src + k) : src[k]; };
    if (lim == 0) return;
    const uint32_t Wu = (uint32_t)W;
    // first marker: the directory's entry, whose runs cover the tile's first word, so its fill
    // starts d = ts - pos >= 0 words before the tile (both < 2^32: 32-bit arithmetic throughout)
    uint64_t mk = load(0);
    uint32_t dirty = (uint32_t)(mk >> 33);
    uint32_t carry;  // -dirty pending at the next marker's start (where this marker's literals end)
    uint32_t rel;
    {
        const uint32_t run = (uint32_t)(mk >> 1);
        const uint32_t d = (uint32_t)ts - pos;
        // tile-relative ends of the fill and of the literals, clamped to W (exact below W)
        uint32_t fe, de;
        if (run >= d) {
            fe = min(run - d, Wu);
            de = min(fe + min(dirty, Wu), Wu);
        } else {
            fe = 0u;
            de = min(dirty - (d - run), Wu);  // > 0: the marker covers word ts
        }
        const uint32_t ones = ((uint32_t)mk & 1u) && fe ? 1u : 0u;
        const bool lit = de > fe;
        atomicAdd(&cnt[ones ? 0u : dummy], ones);
        const uint32_t at_fe = (lit ? 0x10000u : 0u) - ones;
        atomicAdd(&cnt[at_fe ? fe : dummy], at_fe);
        if (de >= Wu) return;
        carry = lit ? 0xFFFF0000u : 0u;
        rel = de;
    }
    uint32_t i = 1 + dirty;
    while (i < lim) {
        mk = load(i);
        const uint32_t hi = (uint32_t)(mk >> 32);
        dirty = hi >> 1;
        const uint32_t run = min((uint32_t)(mk >> 1), Wu);
        // a zero-length one-fill adds +1 and -1 at the same word; an update at fe = W lands in
        // the sentinel slot past the tile (both cheaper than testing for them)
        const uint32_t ones = (uint32_t)mk & 1u;
        const uint32_t fe_raw = rel + run;       // <= 2W
        const uint32_t de_raw = fe_raw + dirty;  // < 2^32: dirty < 2^31
        const uint32_t fe = min(fe_raw, Wu);
        const uint32_t litv = hi >= 2u ? 0x10000u : 0u;  // the marker has literals
        // two reductions per marker: (previous literals end | this one-fill starts) at rel,
        // (this one-fill ends | this marker's literals start) at fe
        const uint32_t at_rel = carry + ones;
        const uint32_t at_fe = litv - ones;
        // byte offsets as index * four (runtime 4): IMAD on the FMA pipe instead of an ALU LEA
        // an empty update adds 0 to its real slot (rare on C4: markers are literal groups)
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + rel * four), at_rel);
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + fe * four), at_fe);
        carry = 0u - litv;
        if (de_raw >= Wu) return;  // the pending literal end lies past the tile
        rel = de_raw;
        i += 1 + dirty;
    }
    if (carry) atomicAdd(&cnt[rel], carry);  // stream ended inside the tile
}


// K4: phases A and B.  A warp's lanes are spread over kWT consecutive tiles of kWS = 32 / kWT
// streams (until the end of round 2: one tile of 32 streams, one bulk copy per lane).  The
// segments a stream contributes to consecutive tiles are contiguous in the stream, so one
// TMA bulk copy stages the segments of kWT lanes (kWS copies per warp and batch instead of
// 32: the copies' operands must be warp-uniform, and ptxas issues per-lane copies in a
// ten-instruction ELECT / R2UR / UBLKCP loop that was a third of the kernel's instructions),
// and the copies carry no per-segment alignment padding.  Each lane walks one (stream, tile)
// slice from the warp's private pool with two shared-memory reductions per marker, into its
// tile's difference array; the CTA holds kWT arrays and then runs phase B on all of them.  A
// batch whose segments overflow the pool walks the rest from HBM.  C4, kernel time: one tile
// per CTA 0.647 ms; kWT = 8 (2 or 3 CTAs/SM) 0.67; kWT = 4, 256 threads, 3 CTAs/SM 0.570;
// kWT = 2 at 4 x 256 or 7 x 128 threads per SM the same; 608-word pools (overflows) 0.68.
#ifndef BQ_K4W_TN
#define BQ_K4W_TN 4
#endif
#ifndef BQ_K4W_NT
#define BQ_K4W_NT 256
#endif
#ifndef BQ_K4W_POOL
#define BQ_K4W_POOL 704
#endif
#ifndef BQ_K4W_MINB
#define BQ_K4W_MINB 3
#endif
constexpr int kWT = BQ_K4W_TN;              // tiles per CTA (a power of two <= 32)
constexpr int kWS = 32 / kWT;               // streams per warp and batch
constexpr int kWThreads = BQ_K4W_NT;
constexpr int kWPool = BQ_K4W_POOL;         // staging words per warp (single-buffered)
constexpr int kWStride = kRleTile + 12 + (kWS > 8 ? 8 : 0);  // words per tile array: [0, W) counts, W sentinel, W + 1 + j dummies
static_assert((kWT & (kWT - 1)) == 0 && kWT <= 32 && kWS <= 16, "lanes = kWS streams x kWT tiles");
constexpr size_t kWCntBytes = (size_t)kWT * kWStride * 4;
constexpr size_t kWBarBytes = (size_t)(kWThreads / 32) * 8;
constexpr size_t kWPoolBytes = (size_t)(kWThreads / 32) * kWPool * 8;
constexpr size_t kWideSmem = kWCntBytes + kWBarBytes +
                             (kWPoolBytes > (size_t)kWT * kRleTile * 2 ? kWPoolBytes : (size_t)kWT * kRleTile * 2);

__global__ void __launch_bounds__(kWThreads, BQ_K4W_MINB) rle_count_kernel(const __grid_constant__ RleCountArgs a) {
    constexpr int NT = kWThreads, NW = NT / 32;
    extern __shared__ __align__(16) uint8_t rle_smem[];
    uint32_t *cnt_all = reinterpret_cast<uint32_t *>(rle_smem);  // kWT packed difference arrays
    uint64_t *bars = reinterpret_cast<uint64_t *>(rle_smem + kWCntBytes);
    uint8_t *region = rle_smem + kWCntBytes + kWBarBytes;  // phase A: warp pools; phase B: undecided list
    __shared__ uint32_t n_und[kWT], todo_slot[kWT];
    __shared__ uint32_t wsum_all[kWT * NW], wreach_all[kWT * NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int li = lane % kWT, lj = lane / kWT;  // this lane's tile within the CTA, stream within the batch
    const int n = a.n;
    const uint32_t first = blockIdx.x * (uint32_t)kWT;              // within the launch
    const uint32_t ntl = min((uint32_t)kWT, a.tile_cnt - first);    // tiles this CTA covers
    const uint32_t tile = a.tile_off + first + (uint32_t)li;        // directory row
    const bool tvalid = (uint32_t)li < ntl;
    const uint64_t ts = (uint64_t)(a.tile0 + tile) * kRleTile;
    const int width = tvalid ? (int)(min(ts + (uint64_t)kRleTile, a.total_words) - ts) : 0;

    for (int k = tid; k < kWT * kWStride; k += NT) cnt_all[k] = 0u;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + warp);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;\n" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // ---- A: run sweep over markers only -> the tiles' difference arrays ---------------
    {
        uint32_t *cnt = cnt_all + (size_t)li * kWStride;
        uint64_t *pool = reinterpret_cast<uint64_t *>(region) + (size_t)warp * kWPool;
        const uint32_t pool_s = (uint32_t)__cvta_generic_to_shared(pool);
        struct Pre {
            uint2 e;
            uint32_t nx;
            uint64_t L;
            const uint64_t *p;
        };
        const int nbatch = (n + kWS - 1) / kWS;
        auto fetch = [&](int b, Pre &q) {
            q.e = make_uint2(0u, 0u);
            q.nx = 0;
            q.L = 0;
            q.p = nullptr;
            const int st = b * kWS + lj;
            if (b < nbatch && st < n && tvalid) {
                q.L = a.lens[st];
                q.e = a.dir[(size_t)tile * n + st];
                q.nx = a.dir[(size_t)(tile + 1) * n + st].x;
                q.p = a.ptrs[st];
            }
        };
        Pre q;
        fetch(warp, q);
        uint32_t parity = 0;
        for (int b = warp; b < nbatch; b += NW) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of the last batch before TMA writes
            // this lane's slice: stream words [lo, hi) = directory marker .. the marker covering the tile's end
            const bool have = q.e.x < q.L;
            const uint32_t lo = have ? q.e.x : 0xFFFFFFFFu;
            uint32_t hi = have ? (uint32_t)min((uint64_t)(q.nx == 0xFFFFFFFFu ? q.L : q.nx) + 1, q.L) : 0u;
            // the batch's stream: [glo, ghi) covers its kWT slices (rows are monotone in the tile)
            const uint32_t glo = __shfl_sync(0xffffffffu, lo, lj * kWT);
#pragma unroll
            for (int o = 1; o < kWT; o <<= 1) hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            const uint64_t *gp = q.p;  // the batch's stream: the same pointer in every valid lane of the group
            uint32_t len = 0;
            uintptr_t b0 = 0;
            if (glo < hi) {
                b0 = reinterpret_cast<uintptr_t>(gp + glo) & ~(uintptr_t)15;
                const uintptr_t b1 = (reinterpret_cast<uintptr_t>(gp + hi) + 15) & ~(uintptr_t)15;
                len = (uint32_t)((b1 - b0) / 8);
            }
            // pool offsets: prefix sum of the groups' lengths (carried by their first lanes)
            const uint32_t off = warp_incl_scan_u32(li == 0 ? len : 0u, lane) - len;
            const bool staged = len && off + len <= (uint32_t)kWPool && a.debug < 2;
            if (li == 0 && staged) {
                const uint32_t bytes = len * 8;
                asm volatile(
                    "{\n\t.reg .b64 st;\n\t"
                    "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
                    "r"(bytes)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        pool_s + off * 8u),
                    "l"(b0), "r"(bytes), "r"(bar)
                    : "memory");
            } else {
                asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
            }
            const uint64_t *g = q.p + q.e.x;
            const uint32_t lim = have ? (uint32_t)(q.L - q.e.x) : 0u;
            const uint32_t pos = q.e.y;
            const uint32_t soff = off + (uint32_t)((reinterpret_cast<uintptr_t>(g) - b0) / 8);
            fetch(b + NW, q);
            {
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                        : "=r"(done)
                        : "r"(bar), "r"(parity)
                        : "memory");
                parity ^= 1u;
            }
            if (lim && !a.debug) {
                if (staged)
                    sweep_stream<false>(pool + soff, lim, pos, ts, width, cnt, a.four, (uint32_t)width + 1 + lj);
                else
                    sweep_stream<true>(g, lim, pos, ts, width, cnt, a.four, (uint32_t)width + 1 + lj);
            }
            __syncwarp();
        }
    }
    __syncthreads();

    // ---- B, all of the CTA's tiles between the same barriers: prefix sums, then decide every
    // word the fills decide; C is deferred to K4c.  (Tile by tile it was 4 barrier rounds per
    // tile with 4 words per thread between them.)
    {
        constexpr int kPer = kRleTile / NT;
        uint32_t *warp_sums = wsum_all, *warp_reach = wreach_all;  // [kWT][NW]
        uint32_t local[kWT][kPer], run_sum[kWT], incl[kWT];
#pragma unroll
        for (int i = 0; i < kWT; ++i) {
            const uint32_t *cnt = cnt_all + (size_t)i * kWStride;
            uint32_t rs = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                rs += cnt[tid * kPer + k];
                local[i][k] = rs;
            }
            run_sum[i] = rs;
            incl[i] = warp_incl_scan_u32(rs, lane);
            if (lane == 31) warp_sums[i * NW + warp] = incl[i];
        }
        if (tid < kWT) n_und[tid] = 0;
        __syncthreads();
        uint32_t reach[kWT];
#pragma unroll
        for (int i = 0; i < kWT; ++i) {
            uint32_t *cnt = cnt_all + (size_t)i * kWStride;
            uint32_t warp_off = 0;
            for (int w = 0; w < warp; ++w) warp_off += warp_sums[i * NW + w];
            const uint32_t excl = warp_off + incl[i] - run_sum[i];
            uint32_t r = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const uint32_t c = local[i][k] + excl;
                cnt[tid * kPer + k] = c;
                r = max(r, (c & 0xFFFFu) + (c >> 16));
            }
            r = __reduce_max_sync(0xffffffffu, r);
            if (lane == 0) warp_reach[i * NW + warp] = r;
        }
        __syncthreads();
        unsigned long long pc = 0;
#pragma unroll
        for (int i = 0; i < kWT; ++i) {
            if ((uint32_t)i >= ntl) break;  // block-uniform
            uint32_t r = 0;
            for (int w = 0; w < NW; ++w) r = max(r, warp_reach[i * NW + w]);
            reach[i] = r;
            const uint32_t trow = a.tile_off + first + (uint32_t)i;
            const uint64_t tsi = (uint64_t)(a.tile0 + trow) * kRleTile;
            const int wi = (int)(min(tsi + (uint64_t)kRleTile, a.total_words) - tsi);
            TileDecide d{tsi, wi, a.total_words, a.last_mask, a.accept_bits, a.const_until, a.out,
                         (uint64_t)a.tile0 * kRleTile, a.breaks, a.nbreak};
            pc += tile_decide<NT>(d, cnt_all + (size_t)i * kWStride, reach[i],
                                  reinterpret_cast<uint16_t *>(region) + (size_t)i * kRleTile, &n_und[i]);
        }
        __syncthreads();
        // tiles with undecided words: a slot in K4c's list each, and their scanned counts
        if (tid < (int)ntl && n_und[tid]) {
            const uint32_t slot = atomicAdd(a.todo_count, 1u);
            a.todo[slot] = a.tile_off + first + (uint32_t)tid;
            todo_slot[tid] = slot;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kWT; ++i) {
            if ((uint32_t)i >= ntl || !n_und[i]) continue;  // block-uniform
            uint4 *dst = reinterpret_cast<uint4 *>(a.todo_cnt + (size_t)todo_slot[i] * kRleTile);
            const uint4 *src = reinterpret_cast<const uint4 *>(cnt_all + (size_t)i * kWStride);
            for (int k = tid; k < kRleTile / 4; k += NT) dst[k] = src[k];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pc += __shfl_down_sync(0xffffffffu, pc, o);
        if (lane == 0 && pc && a.popcnt) atomicAdd(a.popcnt, pc);
    }
}

// K4c: phase C of the tiles K4 deferred (the same tile_resolve, one CTA of kResolveThreads
// per tile, streams walked one per thread four at a time, and a larger literal-address
// buffer than K4's pools leave room for).  A persistent grid takes the deferred tiles in
// order; the decided words of these tiles were written by K4.
#ifndef BQ_K4C_THREADS
#define BQ_K4C_THREADS 1024  // 512: T = 10 / 20 first evaluations 3.70 / 6.59 ms against 3.55 / 6.19 (C4)
#endif
#ifndef BQ_K4C_SLOTS
#define BQ_K4C_SLOTS 1024
#endif
constexpr int kResolveThreads = BQ_K4C_THREADS;
constexpr int kResolveSlots = BQ_K4C_SLOTS;
#ifndef BQ_K4C_CAP
#define BQ_K4C_CAP 4096
#endif
constexpr int kResolveCapC = BQ_K4C_CAP;  // literal words per batch (8 bytes each)
// The tile's stream slices (directory marker .. the marker covering the tile's end, literal
// words included) are staged into one CTA-wide pool by TMA bulk copies, one per stream, so
// phase C's marker walks and literal loads read shared memory instead of following ~10-30
// dependent HBM loads per stream; one CTA per SM.  C4 needs ~19.6 k words per tile.
#ifndef BQ_K4C_POOL
#define BQ_K4C_POOL 21504
#endif
#ifndef BQ_K4C_STAGED
#define BQ_K4C_STAGED 1024  // streams with a stage_off entry (the rest walk HBM)
#endif
constexpr int kResolvePool = BQ_K4C_POOL;
constexpr int kResolveStaged = BQ_K4C_STAGED;
static_assert(kResolveStaged % kResolveThreads == 0, "staging plans kResolveStaged / NT streams per thread");
constexpr size_t kResolveFixed = (size_t)(kRleTile + 4) * 4 + tile_resolve_bytes<kResolveSlots, kResolveCapC>() +
                                 (size_t)kRleTile * 2;
constexpr size_t kResolveSmem = kResolveFixed + (size_t)kResolveStaged * 8 + 16 + (size_t)kResolvePool * 8;
static_assert(kResolveFixed % 16 == 0, "pool alignment");

__global__ void __launch_bounds__(kResolveThreads, 1) rle_resolve_kernel(const __grid_constant__ RleCountArgs a) {
    constexpr int NT = kResolveThreads;
    constexpr int kPerT = kResolveStaged / NT;
    extern __shared__ __align__(16) uint8_t rs_smem[];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rs_smem);
    uint8_t *region = rs_smem + (size_t)(kRleTile + 4) * 4;
    uint16_t *undecided = reinterpret_cast<uint16_t *>(region + tile_resolve_bytes<kResolveSlots, kResolveCapC>());
    uint32_t *stage_off = reinterpret_cast<uint32_t *>(rs_smem + kResolveFixed);
    uint32_t *stage_end = stage_off + kResolveStaged;
    uint64_t *bar_p = reinterpret_cast<uint64_t *>(rs_smem + kResolveFixed + (size_t)kResolveStaged * 8);
    uint64_t *pool = reinterpret_cast<uint64_t *>(rs_smem + kResolveFixed + (size_t)kResolveStaged * 8 + 16);
    __shared__ uint32_t n_undecided, stage_tot[NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.n;
    const int nstaged = min(n, kResolveStaged);
    const uint32_t ntodo = *a.todo_count;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(bar_p);
    const uint32_t pool_s = (uint32_t)__cvta_generic_to_shared(pool);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(NT) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;
    unsigned long long pc = 0;
    for (uint32_t k = blockIdx.x; k < ntodo; k += gridDim.x) {
        const uint32_t tile = a.todo[k];
        const uint64_t ts = (uint64_t)(a.tile0 + tile) * kRleTile;
        const uint64_t te = min(ts + (uint64_t)kRleTile, a.total_words);
        const int width = (int)(te - ts);
        if (tid == 0) n_undecided = 0;
        // ---- stage the slices of streams [0, nstaged): thread tid plans streams tid * kPerT + j ----
        uint32_t len[kPerT], head[kPerT], first_w[kPerT], sum = 0;
        uintptr_t src[kPerT];
#pragma unroll
        for (int j = 0; j < kPerT; ++j) {
            const int st = tid * kPerT + j;
            len[j] = 0;
            head[j] = 0;
            first_w[j] = 0;
            src[j] = 0;
            if (st < nstaged && a.debug < 2) {
                const uint64_t L = a.lens[st];
                const uint2 e = a.dir[(size_t)tile * n + st];
                const uint32_t nx = a.dir[(size_t)(tile + 1) * n + st].x;
                if (e.x < L && e.y < te) {
                    const uint64_t *p = a.ptrs[st];
                    const uint64_t hi = min((uint64_t)(nx == 0xFFFFFFFFu ? L : nx) + 1, L);
                    src[j] = reinterpret_cast<uintptr_t>(p + e.x) & ~(uintptr_t)15;
                    const uintptr_t b1 = (reinterpret_cast<uintptr_t>(p + hi) + 15) & ~(uintptr_t)15;
                    len[j] = (uint32_t)((b1 - src[j]) / 8);
                    head[j] = (uint32_t)((reinterpret_cast<uintptr_t>(p + e.x) - src[j]) / 8);
                    first_w[j] = e.x;
                }
            }
            sum += len[j];
        }
        const uint32_t incl = warp_incl_scan_u32(sum, lane);
        if (lane == 31) stage_tot[warp] = incl;
        __syncthreads();
        uint32_t off = incl - sum;
        for (int w = 0; w < warp; ++w) off += stage_tot[w];
        uint32_t bytes = 0;
#pragma unroll
        for (int j = 0; j < kPerT; ++j) {
            const int st = tid * kPerT + j;
            const bool staged = len[j] && off + len[j] <= (uint32_t)kResolvePool;
            stage_off[st] = staged ? off + head[j] : kNotStaged;
            stage_end[st] = first_w[j] - head[j] + len[j];  // may exceed the stream by the alignment word: never read
            if (!staged) len[j] = 0;
            bytes += len[j] * 8;
            off += len[j] ? len[j] : 0;
        }
        // one arrival per thread carrying its copies' bytes, then the copies
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
                     "r"(bytes)
                     : "memory");
        {
            uint32_t o = off;
#pragma unroll
            for (int j = kPerT - 1; j >= 0; --j) {
                o -= len[j];
                if (len[j])
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            pool_s + o * 8u),
                        "l"(src[j]), "r"(len[j] * 8u), "r"(bar)
                        : "memory");
            }
        }
        // meanwhile: the tile's scanned counts and the undecided words, as phase B classified them
        const uint4 *csrc = reinterpret_cast<const uint4 *>(a.todo_cnt + (size_t)k * kRleTile);
        for (int j = tid; j < kRleTile / 4; j += NT) reinterpret_cast<uint4 *>(cnt)[j] = csrc[j];
        __syncthreads();
        for (int j = tid; j < width; j += NT) {
            const uint32_t c = cnt[j];
            const uint32_t ones = c & 0xFFFFu, dirty = c >> 16;
            if (ones + dirty > __ldg(a.const_until + ones)) undecided[atomicAdd(&n_undecided, 1u)] = (uint16_t)j;
        }
        {
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(bar), "r"(parity)
                    : "memory");
            parity ^= 1u;
        }
        __syncthreads();
        TileDecide d{ts, width, a.total_words, a.last_mask, a.accept_bits, a.const_until, a.out,
                     (uint64_t)a.tile0 * kRleTile, a.breaks, a.nbreak};
        pc += tile_resolve<NT, kResolveSlots, kResolveCapC>(
            d, cnt, undecided, n_undecided, region, [&](const uint16_t *slot_of, auto &&add_bits) {
                walk_tiles<BQ_K4_C_ILP>(a, tid, NT, tile, ts, te, pool, stage_off, stage_end, nstaged,
                                        [&](uint64_t, uint64_t, uint32_t, uint64_t ds, uint64_t de, uint64_t lit,
                                            const uint64_t *s) {
                                            const uint64_t lo = max(ds, ts), hi = min(de, te);
                                            for (uint64_t p = lo; p < hi; ++p) {
                                                const uint16_t u = slot_of[p - ts];
                                                if (u != kNoSlot) add_bits(u, s + lit + (p - ds));
                                            }
                                        });
            });
        __syncthreads();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of the pool before the next tile's copies
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_down_sync(0xffffffffu, pc, o);
    if (lane == 0 && pc && a.popcnt) atomicAdd(a.popcnt, pc);
}

}  // namespace bq

using namespace bq;

struct bq_rle_query {
    int device;
    int n;
    uint64_t r_bits, total_words;
    uint64_t w_begin, w_end;  // output word range (w_begin a multiple of kRleTile)
    uint32_t tile0, ntiles;   // its tiles [tile0, tile0 + ntiles); the directory has ntiles + 1 rows
    void *mem;  // ptr table | len table | directory | error words
    const uint64_t **d_ptrs;
    uint64_t *d_lens;
    uint2 *d_dir;
    uint64_t dir_bytes;
    int evals = 0;
    bool sliced_tried = false;
    SlicedLayout sliced;  // tile-sliced layout (K4s), the default derived layout
    // device accept / const_until / breakpoint tables by accept vector: immutable once
    // uploaded, so repeated evaluations (same T) need no allocation or copy
    std::map<std::vector<uint8_t>, CachedTable> tables;
    StreamUses uses;              // caller streams that evaluated this query (destroy waits on them)
    mutable std::mutex build_mu;  // guards evals / sliced_tried / sliced / tables / uses
};

// Validation of streams over a bit_length-0 universe (host walk; valid streams
// hold only empty markers, so they are short in practice).
static int validate_empty_universe(const std::vector<const uint64_t *> &ptrs, const std::vector<uint64_t> &lens) {
    for (size_t i = 0; i < ptrs.size(); ++i) {
        if (!lens[i]) continue;
        std::vector<uint64_t> h(lens[i]);
        cudaError_t e = cudaMemcpy(h.data(), ptrs[i], lens[i] * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_error(e, "stream copy");
        uint64_t k = 0, covered = 0;
        while (k < h.size()) {
            const uint64_t run = (h[k] >> 1) & 0xFFFFFFFFull, dirty = h[k] >> 33;
            ++k;
            covered += run;
            if (dirty) {
                if (k + dirty > h.size())
                    return set_error(BQ_EFORMAT, "stream %zu: marker announces more literal words than present", i);
                k += dirty;
                covered += dirty;
            }
        }
        if (covered) return set_error(BQ_EFORMAT, "stream %zu: encoded words exceed bit_length", i);
    }
    return BQ_OK;
}

extern "C" {

BQ_API int bq_rle_query_create(const bq_rle_span *streams, int n, uint64_t r_bits, int device, bq_rle_query **out) {
    return bq_rle_query_create_range(streams, n, r_bits, 0, UINT64_MAX, device, out);
}

BQ_API int bq_rle_query_create_range(const bq_rle_span *streams, int n, uint64_t r_bits, uint64_t w_begin,
                                     uint64_t w_end, int device, bq_rle_query **out) {
    if (!out) return set_error(BQ_EINPUT, "out is NULL");
    *out = nullptr;
    if (n < 1) return set_error(BQ_EINPUT, "need at least one input bitmap");
    if (n > BQ_MAX_INPUTS) return set_error(BQ_EINPUT, "%d inputs exceed BQ_MAX_INPUTS=%d", n, BQ_MAX_INPUTS);
    if (!streams) return set_error(BQ_EINPUT, "streams is NULL");
    const uint64_t total = word_count(r_bits);
    if (total >= (1ull << 32) - 2)
        return set_error(BQ_EINPUT, "bit_length too large for the RLE directory (< 2^38 - 128 bits)");
    for (int i = 0; i < n; ++i) {
        if (streams[i].n_words >= (1ull << 32) - 2)
            return set_error(BQ_EINPUT, "stream %d longer than 2^32 - 3 words", i);
        if (streams[i].n_words && !streams[i].words) return set_error(BQ_EINPUT, "stream %d is NULL", i);
        if (reinterpret_cast<uintptr_t>(streams[i].words) & 7)
            return set_error(BQ_EINPUT, "stream %d: device words must be 8-byte aligned", i);
    }
    if (w_end > total) w_end = total;
    if (w_begin > w_end) return set_error(BQ_EINPUT, "word range [%llu, %llu) is empty or reversed",
                                          (unsigned long long)w_begin, (unsigned long long)w_end);
    if (w_begin % kRleTile || (w_end % kRleTile && w_end != total))
        return set_error(BQ_EINPUT, "RLE word range bounds must be multiples of %d words (or the end)", kRleTile);
    DeviceGuard dg;
    int rc = dg.set(device);
    if (rc) return rc;
    const uint32_t tile0 = (uint32_t)(w_begin / kRleTile);
    const uint32_t ntiles = (uint32_t)((w_end - w_begin + kRleTile - 1) / kRleTile);
    std::vector<uint64_t> lens(n);
    for (int i = 0; i < n; ++i) lens[i] = streams[i].n_words;
    const size_t tab = (size_t)n * 16;
    const size_t dirb = (size_t)n * (ntiles + 1) * sizeof(uint2);
    const size_t scr_off = (tab + dirb + 255) & ~(size_t)255;
    const size_t bytes = scr_off + (total ? rle_directory_scratch_bytes(lens) : 0);
    bq_rle_query *q = new bq_rle_query();
    q->device = device;
    q->n = n;
    q->r_bits = r_bits;
    q->total_words = total;
    q->w_begin = w_begin;
    q->w_end = w_end;
    q->tile0 = tile0;
    q->ntiles = ntiles;
    q->dir_bytes = dirb;
    // stream-ordered on the legacy stream, like every use below; the build synchronises
    // that stream before returning, so the query is usable from any stream afterwards
    cudaError_t e = pool_alloc_on(reinterpret_cast<void **>(&q->mem), bytes, 0);
    if (e != cudaSuccess) {
        delete q;
        return cuda_error(e, "cudaMalloc(rle directory)");
    }
    char *m = static_cast<char *>(q->mem);
    q->d_ptrs = reinterpret_cast<const uint64_t **>(m);
    q->d_lens = reinterpret_cast<uint64_t *>(m + (size_t)n * 8);
    q->d_dir = reinterpret_cast<uint2 *>(m + tab);
    std::vector<uint64_t> ptab(2 * (size_t)n);  // pointer table then lengths: one copy
    for (int i = 0; i < n; ++i) {
        ptab[i] = reinterpret_cast<uint64_t>(streams[i].words);
        ptab[(size_t)n + i] = lens[i];
    }
    // with a directory to build, the tables go up with its job table (one pinned staging,
    // ordered on the legacy stream before the kernel; the build synchronises before
    // returning, so they are complete before any evaluation reads them)
    if (!total) {
        e = cudaMemcpyAsync(q->d_ptrs, ptab.data(), tab, cudaMemcpyHostToDevice, 0);
        if (e == cudaSuccess) e = cudaStreamSynchronize(0);
        if (e != cudaSuccess) {
            pool_free(q->mem);
            delete q;
            return cuda_error(e, "rle query setup");
        }
    }
    if (total) {  // the directory walk validates every stream whole, whatever the range
        int code = 0;
        uint64_t bad = 0;
        const uint64_t tail_mask = (r_bits % W) ? ((1ull << (r_bits % W)) - 1) : 0ull;
        rc = build_rle_directory(q->d_ptrs, q->d_lens, lens, total, tail_mask, tile0, ntiles + 1, q->d_dir,
                                 m + scr_off, &code, &bad, ptab.data(), q->d_ptrs, tab);
        if (rc || code) {
            pool_free(q->mem);
            delete q;
            if (rc) return rc;
            const unsigned long long b = (unsigned long long)bad;
            if (code == RLE_ERR_TRUNCATED)
                return set_error(BQ_EFORMAT, "stream %llu: marker announces more literal words than present", b);
            if (code == RLE_ERR_BEYOND_R)
                return set_error(BQ_EFORMAT, "stream %llu: set bits at positions >= bit_length", b);
            return set_error(BQ_EFORMAT, "stream %llu: encoded words exceed bit_length", b);
        }
    } else {
        // bit_length 0: no directory, but the streams are still validated as
        // iter_word_segments would (bitmaps.py:196-219): a truncated literal group, or
        // any fill / literal coverage at all (> 0 words), is a FormatError
        std::vector<const uint64_t *> ptrs(n);
        for (int i = 0; i < n; ++i) ptrs[i] = streams[i].words;
        rc = validate_empty_universe(ptrs, lens);
        if (rc) {
            pool_free(q->mem);
            delete q;
            return rc;
        }
    }
    *out = q;
    return BQ_OK;
}

BQ_API void bq_rle_query_destroy(bq_rle_query *q) {
    if (!q) return;
    DeviceGuard dg;
    dg.set(q->device);
    // stream-ordered: the memory returns to the pool once the evaluations already
    // enqueued on the caller's streams are done; no device-wide synchronisation
    pool_free_after(q->mem, q->uses);
    free_sliced(&q->sliced, &q->uses);
    for (auto &kv : q->tables) cached_table_free(kv.second, q->uses);
    q->uses.release();
    delete q;
}

BQ_API uint64_t bq_rle_query_directory_bytes(const bq_rle_query *q) {
    if (!q) return 0;
    std::lock_guard<std::mutex> guard(q->build_mu);
    return q->dir_bytes + q->sliced.bytes;
}

BQ_API uint64_t bq_rle_query_out_words(const bq_rle_query *q) { return q ? q->w_end - q->w_begin : 0; }

BQ_API int bq_rle_query_layout_stats(const bq_rle_query *q, uint64_t *n_markers, uint64_t *n_literals) {
    if (!q || !n_markers || !n_literals) return set_error(BQ_EINPUT, "NULL argument");
    std::lock_guard<std::mutex> guard(q->build_mu);
    *n_markers = q->sliced.n_markers;
    *n_literals = q->sliced.n_literals;
    return BQ_OK;
}

BQ_API int bq_rle_query_layout_events(const bq_rle_query *q, uint64_t *n_events) {
    if (!q || !n_events) return set_error(BQ_EINPUT, "NULL argument");
    std::lock_guard<std::mutex> guard(q->build_mu);
    *n_events = q->sliced.n_events;
    return BQ_OK;
}


static void note_use(bq_rle_query *q, cudaStream_t s) {
    std::lock_guard<std::mutex> guard(q->build_mu);
    q->uses.note(s);
}

static int rle_eval(bq_rle_query *q, const std::vector<uint8_t> &acc, uint64_t *d_out, unsigned long long *d_popcnt,
                    void *stream) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    if (q->ntiles && !d_out) return set_error(BQ_EINPUT, "d_out is NULL");
    if (reinterpret_cast<uintptr_t>(d_out) & 15) return set_error(BQ_EINPUT, "d_out must be 16-byte aligned");
    DeviceGuard dg;
    int rc = dg.set(q->device);
    if (rc) return rc;
    if (!q->ntiles) return BQ_OK;
    const int n = q->n;
    // accept bits and const_until table (host, O(n))
    const size_t nbits_words = (size_t)(n + 1 + 31) / 32;
    std::vector<uint32_t> host(nbits_words + (size_t)n + 1, 0u);
    for (int k = 0; k <= n; ++k)
        if (acc[k]) host[k >> 5] |= 1u << (k & 31);
    uint32_t *cu = host.data() + nbits_words;
    cu[n] = (uint32_t)n;
    for (int k = n - 1; k >= 0; --k) cu[k] = (acc[k] == acc[k + 1]) ? cu[k + 1] : (uint32_t)k;
    // breakpoints b (accept[b] != accept[b - 1]): phase C decides 64 bits per comparison
    constexpr int kMaxTileBreaks = 64;
    std::vector<uint32_t> brk;
    for (int b = 1; b <= n; ++b)
        if (acc[b] != acc[b - 1]) brk.push_back((uint32_t)b);
    const int nbreak = brk.size() <= (size_t)kMaxTileBreaks ? (int)brk.size() : -1;
    const size_t brk_off = host.size();
    if (nbreak > 0) host.insert(host.end(), brk.begin(), brk.end());
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void *d_tab = nullptr;
    bool owned = false;  // a table outside the query's cache, freed after this launch
    const size_t bytes = host.size() * 4;
    cudaError_t e = cudaSuccess;
    {
        constexpr size_t kMaxTables = 64;
        std::lock_guard<std::mutex> guard(q->build_mu);
        auto it = q->tables.find(acc);
        if (it != q->tables.end()) {
            d_tab = it->second.p;
            e = cached_table_use(it->second, s);  // ordered after its upload, whichever stream did it
            if (e != cudaSuccess) return cuda_error(e, "accept table wait");
        } else if (q->tables.size() < kMaxTables) {
            CachedTable t;
            e = cached_table_upload(t, host.data(), bytes, s);
            if (e != cudaSuccess) {
                if (t.p) pool_free(t.p);
                if (t.ready) cudaEventDestroy(t.ready);
                return cuda_error(e, "accept table upload");
            }
            d_tab = t.p;
            q->tables.emplace(acc, t);
        }
    }
    if (!d_tab) {
        owned = true;
        e = cudaMallocAsync(&d_tab, bytes, s);
        if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(accept)");
        e = cudaMemcpyAsync(d_tab, host.data(), bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) {
            cudaFreeAsync(d_tab, s);
            return cuda_error(e, "cudaMemcpyAsync(accept)");
        }
    }
    auto release = [&] {
        if (owned) cudaFreeAsync(d_tab, s);
    };
    RleCountArgs a;
    a.ptrs = q->d_ptrs;
    a.lens = q->d_lens;
    a.dir = q->d_dir;
    a.n = n;
    a.total_words = q->total_words;
    a.tile0 = q->tile0;
    a.last_mask = (q->r_bits % W) ? ((1ull << (q->r_bits % W)) - 1) : ~0ull;
    a.accept_bits = static_cast<const uint32_t *>(d_tab);
    a.const_until = static_cast<const uint32_t *>(d_tab) + nbits_words;
    a.breaks = static_cast<const uint32_t *>(d_tab) + brk_off;
    a.nbreak = nbreak;
    a.out = d_out;
    a.popcnt = d_popcnt;
    a.four = 4;
    static const char *dbg = getenv("BQ_RLE_DEBUG");
    a.debug = dbg ? atoi(dbg) : 0;
    // Tile-sliced layout policy (BQ_RLE_SLICED): "0" never; "1" build at the first
    // evaluation; default: build at the second one, so a one-shot query does not pay
    // the re-encoding and a reused query (cache hit, several thresholds) gets K4s.
    const char *tenv = getenv("BQ_RLE_SLICED");
    const int sliced_mode = tenv ? atoi(tenv) : 2;
    SlicedLayout sliced;
    {
        // evaluations of one query may come from several host threads (inputs are shared,
        // SPEC.md:269-270): the layout is built once, under the query's lock
        std::lock_guard<std::mutex> guard(q->build_mu);
        ++q->evals;
        if (sliced_mode && !q->sliced_tried && q->evals >= sliced_mode) {
            q->sliced_tried = true;
            e = cudaStreamSynchronize(s);  // the build runs on the legacy stream
            if (e != cudaSuccess) {
                release();
                return cuda_error(e, "cudaStreamSynchronize");
            }
            rc = build_sliced(q->d_ptrs, q->d_lens, q->d_dir, n, q->tile0, q->ntiles, &q->sliced);
            if (rc) {
                release();
                return rc;
            }
        }
        sliced = q->sliced;
    }
    if (sliced.mem && sliced_mode) {
        SlicedEval se{};
        se.n = n;
        se.total_words = q->total_words;
        se.tile0 = q->tile0;
        se.ntiles = q->ntiles;
        se.last_mask = a.last_mask;
        se.accept_bits = a.accept_bits;
        se.const_until = a.const_until;
        se.breaks = a.breaks;
        se.nbreak = a.nbreak;
        se.out = d_out;
        se.popcnt = d_popcnt;
        se.debug = a.debug;
        rc = launch_sliced(sliced, se, s);
        release();
        if (rc == BQ_OK) note_use(q, s);
        return rc;
    } else {
        // K4 (phases A, B), then K4c over the tiles it deferred (scratch in stream order), in
        // chunks of at most kChunk tiles so the deferred counts need at most 256 MB
        const char *chenv = getenv("BQ_K4_CHUNK");  // tests: small chunks
        const uint32_t kChunk = chenv && atoi(chenv) > 0 ? (uint32_t)atoi(chenv) : 65536u;
        const uint32_t chunk = std::min<uint32_t>(q->ntiles, kChunk);
        const size_t b_todo = (((size_t)chunk + 1) * 4 + 255) & ~(size_t)255;
        void *scr = nullptr;
        e = pool_alloc_on(&scr, b_todo + (size_t)chunk * kRleTile * 4, s);
        if (e == cudaSuccess) {
            a.todo_count = static_cast<uint32_t *>(scr);
            a.todo = a.todo_count + 1;
            a.todo_cnt = reinterpret_cast<uint32_t *>(static_cast<char *>(scr) + b_todo);
            e = cudaFuncSetAttribute(rle_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideSmem);
        }
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(rle_resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResolveSmem);
        static int per_sm = 0;
        if (e == cudaSuccess && !per_sm) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rle_resolve_kernel, kResolveThreads, kResolveSmem);
            per_sm = std::max(per_sm, 1);
        }
        for (uint32_t t0 = 0; e == cudaSuccess && t0 < q->ntiles; t0 += chunk) {
            const uint32_t nt = std::min<uint32_t>(chunk, q->ntiles - t0);
            a.tile_off = t0;
            a.tile_cnt = nt;
            e = cudaMemsetAsync(a.todo_count, 0, 4, s);
            if (e == cudaSuccess) {
                rle_count_kernel<<<(nt + kWT - 1) / kWT, kWThreads, kWideSmem, s>>>(a);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) {
                const unsigned grid = (unsigned)std::min<uint64_t>(nt, (uint64_t)sm_count() * per_sm);
                rle_resolve_kernel<<<grid, kResolveThreads, kResolveSmem, s>>>(a);
                e = cudaGetLastError();
            }
        }
        if (scr) cudaFreeAsync(scr, s);
    }
    if (e != cudaSuccess) {
        release();
        return cuda_error(e, "cudaFuncSetAttribute(rle_count_kernel)");
    }
    e = cudaGetLastError();
    release();
    if (e != cudaSuccess) return cuda_error(e, "rle_count_kernel launch");
    note_use(q, s);
    return BQ_OK;
}

BQ_API int bq_rle_query_sweep_stats(bq_rle_query *q, int t, uint64_t *h_stats, void *stream) {
    if (!q || !h_stats) return set_error(BQ_EINPUT, "NULL argument");
    if (t < 0 || t > q->n) return set_error(BQ_EINPUT, "threshold %d outside [0, %d]", t, q->n);
    if (q->w_begin != 0 || q->w_end != q->total_words)
        return set_error(BQ_EINPUT, "sweep stats describe the whole sweep: the query must cover all words");
    DeviceGuard dg;
    int rc = dg.set(q->device);
    if (rc) return rc;
    for (int k = 0; k < 6; ++k) h_stats[k] = 0;
    if (!q->total_words) return BQ_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = rle_sweep_stats(q->d_ptrs, q->d_lens, q->d_dir, q->n, q->ntiles, q->total_words, t, h_stats, s);
    if (rc == BQ_OK) note_use(q, s);
    return rc;
}

BQ_API int bq_rle_query_threshold(bq_rle_query *q, int t, uint64_t *d_out, unsigned long long *d_popcnt, void *stream) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    if (t < 1 || t > q->n) return set_error(BQ_EINPUT, "threshold %d outside [1, %d]", t, q->n);  // runmerge.py:201-202
    std::vector<uint8_t> acc(q->n + 1);
    for (int k = 0; k <= q->n; ++k) acc[k] = k >= t;
    return rle_eval(q, acc, d_out, d_popcnt, stream);
}

BQ_API int bq_rle_query_symmetric(bq_rle_query *q, const uint8_t *h_accept, uint64_t *d_out,
                                  unsigned long long *d_popcnt, void *stream) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    if (!h_accept) return set_error(BQ_EINPUT, "accept vector is NULL");
    std::vector<uint8_t> acc(h_accept, h_accept + q->n + 1);
    for (auto &v : acc) v = v ? 1 : 0;
    return rle_eval(q, acc, d_out, d_popcnt, stream);
}

}  // extern "C"
