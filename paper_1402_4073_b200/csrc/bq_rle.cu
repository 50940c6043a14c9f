// K3/K4: threshold and symmetric queries over EWAH-style run-length-encoded
// bitmaps, decoded on the device (sm_100a).
//
// Stream format (reference bitmaps.py:27-40): a marker word
//   bit 0 = fill bit, bits 1-32 = fill run (words), bits 33-63 = literal count
// followed by that many literal ("dirty") words; coverage shorter than
// ceil(r/64) words is an implicit zero tail (bitmaps.py:215-219).
//
// K3 the tile directory, once per query object (inputs are immutable):
//   K3a rle_chain_kernel -- one warp per stream follows the marker chain in
//   32-word windows (pointer doubling + warp OR-reductions find a window's
//   markers; windows are cp.async-staged ahead; dirty runs longer than the ring
//   are skipped unread) and keeps per window only its marker mask and start
//   position.  K3b rle_dirfill_kernel -- every window in parallel: marker word
//   positions by a warp prefix sum, the validation of
//   RleBitmap.iter_word_segments (:210-217; FormatError), and a directory entry
//   (marker index, run start) for every tile boundary a marker's runs cover.
//
// K4 rle_count_kernel -- one CTA per tile of kTileWords output words, the
//   per-tile form of cdom's run sweep (runmerge.py:198-299):
//   A. each thread walks whole streams from their directory entry, reading
//      only marker words; one-fill and dirty runs become +1/-1 entries of a
//      packed shared-memory difference array (ones in bits 0-15, dirty in
//      16-31), so a prefix scan yields k_w (one-fills) and d_w (dirty inputs)
//      for every word w;
//   B. w is decided from (k_w, d_w) alone when accept[] is constant on
//      [k_w, k_w + d_w] (cdom's three cases) -- the common
//      case -- and written directly;
//   C. only for undecided words are the dirty literals read: a second walk
//      adds their bits into per-word shared-memory bit counters, then
//      accept[k_w + count_b] decides each bit (dirty_segment_solver's "scan"
//      branch, runmerge.py:99-125).
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

constexpr int kSlotsPerBatch = 512;   // undecided words resolved per phase-C pass
constexpr int kStagedThreads = 128;     // staged K4: 4 warps, each with a private pool
#ifndef BQ_K4_POOL
#define BQ_K4_POOL 768
#endif
#ifndef BQ_K4_MINB
#define BQ_K4_MINB 4
#endif
constexpr int kPoolWords = BQ_K4_POOL;  // words per warp pool half (two halves: double buffer);
                                        // C4 needs ~613 words per 32 streams on average, 760 at p99
constexpr size_t kCntBytes = (size_t)(kRleTile + 36) * 4 + 16 * 16;  // + sentinel, 32 per-lane dummies, mbarriers

constexpr size_t kPoolBytes = (size_t)(kStagedThreads / 32) * 2 * kPoolWords * 8;
constexpr size_t kPhaseCBytes = tile_resolve_bytes<kSlotsPerBatch>() + (size_t)kRleTile * 2;  // + undecided list
constexpr size_t kRegionBytes = kPoolBytes > kPhaseCBytes ? kPoolBytes : kPhaseCBytes;

inline size_t rle_smem_bytes() {
    return kCntBytes + kRegionBytes;
}

enum { RLE_ERR_TRUNCATED = 1, RLE_ERR_OVERLONG = 2, RLE_ERR_BEYOND_R = 3 };

struct RleDirArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    int n;
    uint64_t total_words;  // ceil(r/64)
    uint64_t tail_mask;    // valid bits of the last word when r % 64 != 0, else 0
    uint32_t tile0;        // first tile of the query's word range
    uint32_t nrows;        // directory rows: the range's tiles + 1 (the boundary after its last tile)
    uint2 *dir;            // [nrows][n]: (marker index, run start word); tile-major so a K4 CTA reads one row
    int *err;              // first error code
    unsigned long long *err_stream;
};

__device__ __forceinline__ void rle_fail(const RleDirArgs &a, int code, int stream) {
    if (atomicCAS(a.err, 0, code) == 0) atomicExch(a.err_stream, (unsigned long long)stream);
}

// K3: one warp per stream.  The stream is read in 32-word windows aligned to its
// start, so window loads do not wait for the marker chain: the next window is
// loaded while the current one is decoded (a dirty group reaching past the next
// window jumps straight to the window of the next marker, skipping literals
// unread).  Inside a window, the markers on the chain from every possible entry
// are found at once by pointer jumping; following the chain is a lookup per
// window; marker word positions come from a warp prefix sum in K3b.
constexpr int kDirAhead = 14;  // windows in flight ahead of the one being decoded
constexpr int kDirRing = 16;  // ring slots per warp (> kDirAhead: consumed slots are reused late)
#ifndef BQ_CHAIN_GROUP
#define BQ_CHAIN_GROUP 4
#endif
constexpr int kChainGroup = BQ_CHAIN_GROUP;  // K3a: windows whose chain tables are computed together

// K3a: the sequential part of the directory -- one warp per stream follows its
// marker chain window by window (windows copied into a per-warp ring by per-lane
// cp.async, kDirAhead ahead; a literal group reaching past the ring restarts it
// at the next marker, so long dirty runs are skipped unread).  The chain's
// dependency from window to window is kept short: for every window the warp
// first computes, for all 32 possible entry lanes at once, where the chain from
// that entry leaves the window, which markers it passes and the words they cover
// (pointer jumping: five levels, each combining a lane's aggregate with the one at
// its successor), which does not depend on the actual entry; several windows'
// tables are computed interleaved (kChainGroup windows).  Following the chain is then a lookup (a
// shuffle from the entry lane) per window.  Only two facts per window are kept:
// its marker mask and the word position where its first marker's fill starts.
// Everything else -- marker positions, validation, directory rows -- is K3b, in
// parallel over all windows.
struct ChainTable {
    uint32_t m;   // markers on the chain from this lane, within the window
    uint32_t nx;  // where the chain leaves: window-relative index of its next marker (>= 32, or a lane past L)
};

// This lane's entry of a window's chain table (word w at index bc + lane, valid:
// bc + lane < L).
__device__ __forceinline__ ChainTable chain_table(uint64_t w, bool valid, int lane) {
    ChainTable t;
    t.m = valid ? 1u << lane : 0u;
    t.nx = valid ? (uint32_t)lane + 1u + (uint32_t)(w >> 33) : (uint32_t)lane;  // dirty < 2^31
    return t;
}

__device__ __forceinline__ void chain_jump(ChainTable &t, int lane) {
    const bool on = t.nx < 32u;
    const int src = on ? (int)t.nx : lane;
    const uint32_t m = __shfl_sync(0xffffffffu, t.m, src);
    const uint32_t nx = __shfl_sync(0xffffffffu, t.nx, src);
    t.m |= on ? m : 0u;
    t.nx = on ? nx : t.nx;
}

// Words covered by the fills and literal groups of the window's markers in `reach`
// (each span < 2^40: the two 24-bit-split sums stay exact).
__device__ __forceinline__ uint64_t chain_span(uint64_t w, uint32_t reach, int lane) {
    const uint64_t span = ((reach >> lane) & 1u) ? ((w >> 1) & 0xFFFFFFFFull) + (w >> 33) : 0ull;
    const uint32_t lo = __reduce_add_sync(0xffffffffu, (uint32_t)(span & 0xFFFFFFu));
    const uint32_t hi = __reduce_add_sync(0xffffffffu, (uint32_t)(span >> 24));
    return ((uint64_t)hi << 24) + lo;
}

__global__ void __launch_bounds__(128) rle_chain_kernel(const __grid_constant__ RleDirArgs a, const uint64_t *wbase,
                                                        uint32_t *wreach, uint64_t *wpos) {
    __shared__ uint64_t ring_all[4][kDirRing][32];
    const int lane = threadIdx.x & 31;
    const int stream = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (stream >= a.n) return;
    uint64_t(*ring)[32] = ring_all[threadIdx.x >> 5];
    const uint64_t *s = a.ptrs[stream];
    const uint64_t L = a.lens[stream];
    uint2 *dir = a.dir + stream;  // stride n between tiles
    const uint64_t wb = wbase[stream];
    auto issue = [&](uint64_t q) {
        const uint64_t idx = q * 32 + lane;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[q % kDirRing][lane]);
        const uint64_t *src = s + (idx < L ? idx : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(idx < L ? 8u : 0u)
                     : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    constexpr int G = kChainGroup;  // windows whose tables are computed per iteration
    uint64_t k = 0;     // first window of the group being decoded
    uint64_t next = 0;  // stream index of the next marker
    uint64_t pos = 0;   // word position where its fill run starts
    for (int q = 0; q < kDirAhead; ++q) issue(q);
    while (next < L) {
        const uint64_t kk = next / 32;
        if (kk + G - 1 >= k + kDirAhead) {  // a long literal group: restart the pipeline at the next marker
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            k = kk;
            for (int q = 0; q < kDirAhead; ++q) issue(k + q);
        } else {
            for (; k < kk; ++k) issue(k + kDirAhead);  // windows of literals only
        }
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kDirAhead - G) : "memory");
        // tables of windows k .. k + G - 1 (independent of the entry; interleaved)
        const uint64_t bc0 = k * 32;
        uint64_t w[G];
        ChainTable t[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            w[g] = ring[(k + g) % kDirRing][lane];
            t[g] = chain_table(w[g], bc0 + 32 * g + lane < L, lane);
        }
#pragma unroll
        for (int level = 0; level < 5; ++level)
#pragma unroll
            for (int g = 0; g < G; ++g) chain_jump(t[g], lane);
        // follow the chain through the group while it enters the next window
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint64_t bc = bc0 + 32 * g;
            if (g > 0 && !(next < bc + 32 && next < L)) break;  // g == 0 holds the entry; later ones have next >= bc
            const int e = (int)(next - bc);
            const uint32_t reach = __shfl_sync(0xffffffffu, t[g].m, e);
            const uint32_t nx = __shfl_sync(0xffffffffu, t[g].nx, e);
            if (lane == 0) {
                wreach[wb + k + g] = reach;
                wpos[wb + k + g] = pos;
            }
            pos += chain_span(w[g], reach, lane);
            next = bc + nx;
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    // tiles past the encoded coverage: stream exhausted, implicit zero tail
    const uint64_t t0 = max((pos + kRleTile - 1) / kRleTile, (uint64_t)a.tile0);
    for (uint64_t t = t0 + lane; t < (uint64_t)a.tile0 + a.nrows; t += 32)
        dir[(t - a.tile0) * a.n] = make_uint2((uint32_t)L, (uint32_t)pos);
}

// K3b: every window with markers, in parallel (grid.y = stream): marker word
// positions by a warp prefix sum from the window's start position, validation as
// RleBitmap.iter_word_segments / decompress (bitmaps.py:196-219, :428-431), and
// the directory row of every tile boundary a marker's runs cover.
__global__ void __launch_bounds__(128) rle_dirfill_kernel(const __grid_constant__ RleDirArgs a, const uint64_t *wbase,
                                                          const uint32_t *wreach, const uint64_t *wpos) {
    const int lane = threadIdx.x & 31;
    const int stream = blockIdx.y;
    const uint64_t *s = a.ptrs[stream];
    const uint64_t L = a.lens[stream];
    uint2 *dir = a.dir + stream;
    const uint64_t nwin = (L + 31) / 32, wb = wbase[stream];
    const uint64_t r0 = (uint64_t)a.tile0 * kRleTile, r1 = (uint64_t)(a.tile0 + a.nrows) * kRleTile;
    const uint64_t stride = (uint64_t)gridDim.x * 4;
    uint64_t k = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    // the next window's mask, position and words are loaded one window ahead
    auto load = [&](uint64_t q, uint32_t &r, uint64_t &p, uint64_t &w) {
        if (q < nwin) {
            r = wreach[wb + q];
            p = wpos[wb + q];
            w = q * 32 + lane < L ? __ldg(s + q * 32 + lane) : 0ull;
        }
    };
    uint32_t r_n = 0;
    uint64_t p_n = 0, w_n = 0;
    load(k, r_n, p_n, w_n);
    for (; k < nwin; k += stride) {
        const uint32_t reach = r_n;
        const uint64_t pos = p_n, w = w_n;
        load(k + stride, r_n, p_n, w_n);
        if (!reach) continue;  // a window inside a literal group
        const uint64_t idx = k * 32 + lane;
        const uint64_t run = (w >> 1) & 0xFFFFFFFFull;
        const uint64_t dirty = w >> 33;
        const bool is_m = (reach >> lane) & 1u;
        const uint64_t span = is_m ? run + dirty : 0ull;
        uint64_t incl = span;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (!is_m) continue;
        const uint64_t start = pos + incl - span;
        const uint64_t end = start + span;
        if (idx + 1 + dirty > L) rle_fail(a, RLE_ERR_TRUNCATED, stream);
        if (end > a.total_words) rle_fail(a, RLE_ERR_OVERLONG, stream);
        // bits >= r in the last word are invalid (bitmaps.py:70-72 via decompress :428-431)
        if (a.tail_mask && end == a.total_words && span) {
            const uint64_t fe = start + run;
            if (fe == end) {
                if ((w & 1) && run) rle_fail(a, RLE_ERR_BEYOND_R, stream);
            } else if (idx + 1 + dirty <= L && (__ldg(s + idx + dirty) & ~a.tail_mask)) {
                rle_fail(a, RLE_ERR_BEYOND_R, stream);
            }
        }
        // record every tile boundary b with start <= b < end that the range's rows cover
        uint64_t b = max((start + kRleTile - 1) / kRleTile * kRleTile, r0);
        for (; b < end && b < a.total_words && b < r1; b += kRleTile)
            dir[(b / kRleTile - a.tile0) * (uint64_t)a.n] = make_uint2((uint32_t)idx, (uint32_t)start);
    }
}

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
};


// Walk stream `st` across tile [ts, te) from its directory entry; Visit(fs, fe, bit, ds, de, lit)
// is called for each marker whose runs intersect the tile (fill [fs,fe), dirty [ds,de) with the
// first literal at stream index lit).
template <typename Visit>
__device__ __forceinline__ void walk_tile(const RleCountArgs &a, int st, uint32_t tile, uint64_t ts, uint64_t te,
                                          Visit &&visit) {
    const uint64_t *s = a.ptrs[st];
    const uint64_t L = a.lens[st];
    const uint2 e = a.dir[(size_t)tile * a.n + st];
    uint64_t i = e.x, pos = e.y;
    while (i < L && pos < te) {
        const uint64_t mk = __ldg(s + i);
        const uint64_t run = (mk >> 1) & 0xFFFFFFFFull;
        const uint64_t dirty = mk >> 33;
        const uint64_t fe = pos + run, de = fe + dirty;
        if (de > ts) visit(pos, fe, (uint32_t)(mk & 1), fe, de, i + 1, s);
        pos = de;
        i += 1 + dirty;
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
                                             uint32_t *cnt, uint32_t four) {
    auto load = [src](uint32_t k) { return GLOBAL ? __ldg(src + k) : src[k]; };
    if (lim == 0) return;
    const uint32_t Wu = (uint32_t)W;
    const uint32_t dummy = Wu + 1 + (threadIdx.x & 31);  // this lane's slot for empty contributions
    // first marker: its fill starts at or before the tile (64-bit positions)
    uint64_t mk = load(0);
    uint32_t dirty = (uint32_t)(mk >> 33);
    uint32_t carry;  // -dirty pending at the next marker's start (where this marker's literals end)
    uint32_t rel;
    {
        const int64_t fs64 = (int64_t)pos - (int64_t)ts;
        const int64_t fe64 = fs64 + (int64_t)(uint32_t)(mk >> 1);
        const int64_t de64 = fe64 + dirty;
        auto cl = [W](int64_t v) { return (uint32_t)(v < 0 ? 0 : (v > W ? W : v)); };
        const uint32_t fs = cl(fs64), fe = cl(fe64), de = cl(de64);
        const uint32_t ones = ((mk & 1) && fe > fs) ? 1u : 0u;
        const bool lit = de > fe;
        atomicAdd(&cnt[ones ? fs : dummy], ones);
        const uint32_t at_fe = (lit ? 0x10000u : 0u) - ones;
        atomicAdd(&cnt[at_fe ? fe : dummy], at_fe);
        if (de64 >= W) return;
        carry = lit ? 0xFFFF0000u : 0u;
        rel = (uint32_t)de64;
    }
    uint32_t i = 1 + dirty;
    while (i < lim) {
        mk = load(i);
        dirty = (uint32_t)(mk >> 33);
        const uint32_t run = min((uint32_t)(mk >> 1), Wu);
        const uint32_t ones = (uint32_t)(mk & 1) & (run != 0u);
        const uint32_t fe_raw = rel + run;       // <= 2W
        const uint32_t de_raw = fe_raw + dirty;  // < 2^32: dirty < 2^31
        const uint32_t fe = min(fe_raw, Wu);
        const bool lit = (dirty != 0u) & (fe < Wu);
        // two reductions per marker: (previous literals end | this one-fill starts) at rel,
        // (this one-fill ends | this marker's literals start) at fe
        const uint32_t at_rel = carry + ones;
        const uint32_t at_fe = (lit ? 0x10000u : 0u) - ones;
        // byte offsets as index * four (runtime 4): IMAD on the FMA pipe instead of an ALU LEA
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + (at_rel ? rel : dummy) * four), at_rel);
        atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(cnt) + (at_fe ? fe : dummy) * four), at_fe);
        carry = lit ? 0xFFFF0000u : 0u;
        if (de_raw >= Wu) return;  // the pending literal end lies past the tile
        rel = de_raw;
        i += 1 + dirty;
    }
    if (carry) atomicAdd(&cnt[rel], carry);  // stream ended inside the tile
}


// Phase A: warp-private, double-buffered staging.  Lane l of warp w owns stream
// k*NT + 32w + l of batch k.  It computes its stream's segment for this tile
// (directory entry -> marker covering the next tile boundary, widened to 16-byte
// alignment), claims room in the warp's pool with a warp prefix sum, and copies
// the segment with one TMA bulk copy while the previous batch is being walked;
// one mbarrier per pool half, so the warps never meet at a CTA barrier in phase
// A.  A segment that does not fit the pool is walked straight from HBM.
__global__ void __launch_bounds__(kStagedThreads, BQ_K4_MINB) rle_count_kernel(const __grid_constant__ RleCountArgs a) {
    constexpr int NT = kStagedThreads;
    constexpr int kSlots = kSlotsPerBatch;
    extern __shared__ __align__(16) uint8_t rle_smem[];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rle_smem);  // [kRleTile + 4] packed (ones | dirty << 16)
    uint8_t *region = rle_smem + kCntBytes;                  // phase A: warp pools; phases B/C: tile_resolve
    __shared__ uint32_t n_undecided;
    __shared__ uint32_t warp_sums[NT / 32], warp_reach[NT / 32];

    const uint32_t tile = blockIdx.x;  // directory row; the tile's words are global
    const uint64_t ts = (uint64_t)(a.tile0 + tile) * kRleTile;
    const uint64_t te = min(ts + (uint64_t)kRleTile, a.total_words);
    const int width = (int)(te - ts);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int n = a.n;

    for (int k = tid; k <= kRleTile; k += NT) cnt[k] = 0u;
    if (tid == 0) n_undecided = 0;
    __syncthreads();

    // ---- A: run sweep over markers only -> difference array ------------------
    {
        // directory metadata of a lane's stream in batch k (tile-major rows: coalesced),
        // fetched one batch ahead of use so its latency hides behind a walk
        struct Pre {
            uint2 e;
            uint32_t nx;
            uint64_t L;
            const uint64_t *p;
        };
        auto fetch = [&](int st, Pre &q) {
            q.e = make_uint2(0u, 0u);
            q.L = 0;
            if (st < n) {
                q.L = a.lens[st];
                q.e = a.dir[(size_t)tile * a.n + st];
                q.nx = a.dir[(size_t)(tile + 1) * a.n + st].x;
                q.p = a.ptrs[st];
            }
        };
        uint64_t *pool = reinterpret_cast<uint64_t *>(region) + (size_t)warp * 2 * kPoolWords;
        // one mbarrier per pool half; 32 arrivals (one per lane) + the TMA byte count complete a phase
        uint64_t *bars = reinterpret_cast<uint64_t *>(cnt + kRleTile + 36) + warp * 2;
        const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;\n" ::"r"(bar0) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;\n" ::"r"(bar0 + 8) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
        struct Seg {
            const uint64_t *g;  // global address of the directory marker
            uint32_t lim, pos, off;
            bool staged;
        };
        // Stage batch k's segment of this lane's stream: one TMA bulk copy per lane.
        auto plan = [&](const Pre &q, int k, Seg &sg) {
            sg.lim = 0;
            sg.staged = false;
            uint32_t len = 0;
            uintptr_t b0 = 0;
            if (q.e.x < q.L) {
                const uint64_t next = q.nx == 0xFFFFFFFFu ? q.L : q.nx;
                sg.g = q.p + q.e.x;
                sg.lim = (uint32_t)(q.L - q.e.x);
                sg.pos = q.e.y;
                b0 = reinterpret_cast<uintptr_t>(sg.g) & ~(uintptr_t)15;
                const uintptr_t b1 = (reinterpret_cast<uintptr_t>(q.p + min(next + 1, q.L)) + 15) & ~(uintptr_t)15;
                len = (uint32_t)((b1 - b0) / 8);
            }
            uint32_t incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t off = incl - len;
            const uint32_t bar = bar0 + 8 * (k & 1);
            if (len && incl <= (uint32_t)kPoolWords && a.debug < 2) {
                sg.staged = true;
                sg.off = off + (uint32_t)((reinterpret_cast<uintptr_t>(sg.g) >> 3) & 1);
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pool + (size_t)(k & 1) * kPoolWords + off);
                const uint32_t bytes = len * 8;
                asm volatile(
                    "{\n\t.reg .b64 st;\n\t"
                    "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
                    "r"(bytes)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                    "l"(b0), "r"(bytes), "r"(bar)
                    : "memory");
            } else {
                asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
            }
        };
        auto wait_batch = [&](int k) {
            const uint32_t bar = bar0 + 8 * (k & 1);
            const uint32_t parity = (uint32_t)((k >> 1) & 1);
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(bar), "r"(parity)
                    : "memory");
            }
        };
        const int nk = (n + NT - 1) / NT;
        const int my = warp * 32 + lane;
        // two-batch unrolled pipeline: batch k + 2's metadata lands in q while batch k is
        // walked, and the segment plans alternate between sa / sb (no register rotation
        // that would wait on the metadata loads right after issuing them)
        Seg sa, sb;
        Pre q;
        fetch(my, q);
        plan(q, 0, sa);
        fetch(NT + my, q);
        auto step = [&](int k, Seg &cur, Seg &nxt) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of k-1 before TMA writes
            plan(q, k + 1, nxt);  // k + 1 == nk: nothing to copy, arrive only
            fetch((k + 2) * NT + my, q);
            wait_batch(k);  // every lane's bulk copy for batch k has landed
            if (cur.lim && !a.debug) {
                if (cur.staged)
                    sweep_stream<false>(pool + (size_t)(k & 1) * kPoolWords + cur.off, cur.lim, cur.pos, ts, width, cnt,
                                        a.four);
                else
                    sweep_stream<true>(cur.g, cur.lim, cur.pos, ts, width, cnt, a.four);
            }
            __syncwarp();  // batch k's pool half may be refilled for batch k + 2
        };
        for (int k = 0; k < nk; k += 2) {
            step(k, sa, sb);
            if (k + 1 < nk) step(k + 1, sb, sa);
        }
    }
    __syncthreads();

    // ---- B: prefix sum, then decide every word the fills decide ------------------
    const uint32_t reach = tile_scan<NT>(cnt, warp_sums, warp_reach);
    TileDecide d{ts, width, a.total_words, a.last_mask, a.accept_bits, a.const_until, a.out, (uint64_t)a.tile0 * kRleTile,
                 a.breaks, a.nbreak};
    uint16_t *undecided = reinterpret_cast<uint16_t *>(region + tile_resolve_bytes<kSlots>());
    unsigned long long pc = tile_decide<NT>(d, cnt, reach, undecided, &n_undecided);
    __syncthreads();

    // ---- C: read dirty literals only where the fills leave the outcome open ----
    pc += tile_resolve<NT, kSlots>(d, cnt, undecided, n_undecided, region, [&](const uint16_t *slot_of, auto &&add_bits) {
        for (int st = tid; st < a.n; st += NT) {
            walk_tile(a, st, tile, ts, te,
                      [&](uint64_t, uint64_t, uint32_t, uint64_t ds, uint64_t de, uint64_t lit, const uint64_t *s) {
                          const uint64_t lo = max(ds, ts), hi = min(de, te);
                          for (uint64_t p = lo; p < hi; ++p) {
                              const uint16_t u = slot_of[p - ts];
                              if (u != kNoSlot) add_bits(u, s + lit + (p - ds));
                          }
                      });
        }
    });

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
    std::map<std::vector<uint8_t>, void *> tables;
    StreamUses uses;              // caller streams that evaluated this query (destroy waits on them)
    mutable std::mutex build_mu;  // guards evals / sliced_tried / sliced / tables / uses
};

// The previous K3 (A/B measurements: BQ_RLE_K3=old): K3a walks each stream's chain
// window by window, K3b fills the directory from every window in parallel.
static cudaError_t old_directory(const RleDirArgs &a, const std::vector<uint64_t> &lens, int n, int *d_err) {
    std::vector<uint64_t> wbase(n + 1, 0);
    uint64_t maxwin = 0;
    for (int i = 0; i < n; ++i) {
        const uint64_t nwin = (lens[i] + 31) / 32;
        wbase[i + 1] = wbase[i] + nwin;
        maxwin = std::max(maxwin, nwin);
    }
    const uint64_t nwin_all = wbase[n];
    char *scratch = nullptr;
    cudaError_t e = pool_alloc(reinterpret_cast<void **>(&scratch), (size_t)(n + 1) * 8 + nwin_all * 12 + 16);
    uint64_t *d_wbase = reinterpret_cast<uint64_t *>(scratch);
    uint64_t *d_wpos = d_wbase + n + 1;
    uint32_t *d_wreach = reinterpret_cast<uint32_t *>(d_wpos + nwin_all);
    if (e == cudaSuccess) e = cudaMemcpy(d_wbase, wbase.data(), (size_t)(n + 1) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(d_wreach, 0, nwin_all * 4 + 4);
    if (e == cudaSuccess) {
        rle_chain_kernel<<<(n + 3) / 4, 128>>>(a, d_wbase, d_wreach, d_wpos);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && nwin_all) {
        const unsigned gx = (unsigned)std::min<uint64_t>((maxwin + 3) / 4, 64);
        rle_dirfill_kernel<<<dim3(gx, (unsigned)n), 128>>>(a, d_wbase, d_wreach, d_wpos);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (scratch) pool_free(scratch);
    return e;
}

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
    const size_t tab = (size_t)n * 16;
    const size_t dirb = (size_t)n * (ntiles + 1) * sizeof(uint2);
    const size_t bytes = tab + dirb + 64;
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
    cudaError_t e = pool_alloc(reinterpret_cast<void **>(&q->mem), bytes);
    if (e != cudaSuccess) {
        delete q;
        return cuda_error(e, "cudaMalloc(rle directory)");
    }
    char *m = static_cast<char *>(q->mem);
    q->d_ptrs = reinterpret_cast<const uint64_t **>(m);
    q->d_lens = reinterpret_cast<uint64_t *>(m + (size_t)n * 8);
    q->d_dir = reinterpret_cast<uint2 *>(m + tab);
    int *d_err = reinterpret_cast<int *>(m + tab + dirb);
    unsigned long long *d_err_stream = reinterpret_cast<unsigned long long *>(m + tab + dirb + 8);
    std::vector<const uint64_t *> ptrs(n);
    std::vector<uint64_t> lens(n);
    for (int i = 0; i < n; ++i) {
        ptrs[i] = streams[i].words;
        lens[i] = streams[i].n_words;
    }
    e = cudaMemcpy(q->d_ptrs, ptrs.data(), (size_t)n * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(q->d_lens, lens.data(), (size_t)n * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(d_err, 0, 16);
    if (e != cudaSuccess) {
        pool_free(q->mem);
        delete q;
        return cuda_error(e, "rle query setup");
    }
    if (total) {  // the directory walk validates every stream whole, whatever the range
        RleDirArgs a;
        a.ptrs = q->d_ptrs;
        a.lens = q->d_lens;
        a.n = n;
        a.total_words = total;
        a.tail_mask = (r_bits % W) ? ((1ull << (r_bits % W)) - 1) : 0ull;
        a.tile0 = tile0;
        a.nrows = ntiles + 1;
        a.dir = q->d_dir;
        a.err = d_err;
        a.err_stream = d_err_stream;
        int herr[4] = {0, 0, 0, 0};
        static const char *k3env = getenv("BQ_RLE_K3");
        if (k3env && !strcmp(k3env, "old")) {  // the previous two-kernel form (A/B measurements only)
            e = old_directory(a, lens, n, d_err);
            if (e == cudaSuccess) e = cudaMemcpy(herr, d_err, 16, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                pool_free(q->mem);
                delete q;
                return cuda_error(e, "rle directory (K3)");
            }
        } else {
            uint64_t bad = 0;
            rc = build_rle_directory(q->d_ptrs, q->d_lens, lens, total, a.tail_mask, tile0, ntiles + 1, q->d_dir,
                                     &herr[0], &bad);
            if (rc) {
                pool_free(q->mem);
                delete q;
                return rc;
            }
            herr[2] = (int)(uint32_t)bad;
            herr[3] = (int)(uint32_t)(bad >> 32);
        }
        if (herr[0]) {
            unsigned long long bad = (unsigned long long)(uint32_t)herr[2] | ((unsigned long long)(uint32_t)herr[3] << 32);
            pool_free(q->mem);
            delete q;
            if (herr[0] == RLE_ERR_TRUNCATED)
                return set_error(BQ_EFORMAT, "stream %llu: marker announces more literal words than present", bad);
            if (herr[0] == RLE_ERR_BEYOND_R)
                return set_error(BQ_EFORMAT, "stream %llu: set bits at positions >= bit_length", bad);
            return set_error(BQ_EFORMAT, "stream %llu: encoded words exceed bit_length", bad);
        }
    } else {
        // bit_length 0: no directory, but the streams are still validated as
        // iter_word_segments would (bitmaps.py:196-219): a truncated literal group, or
        // any fill / literal coverage at all (> 0 words), is a FormatError
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
    for (auto &kv : q->tables) pool_free_after(kv.second, q->uses);
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
            d_tab = it->second;
        } else if (q->tables.size() < kMaxTables) {
            e = pool_alloc(reinterpret_cast<void **>(&d_tab), bytes);
            // ordered on the consuming stream, and complete before the table is shared
            // with evaluations on other streams
            if (e == cudaSuccess) e = cudaMemcpyAsync(d_tab, host.data(), bytes, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                if (d_tab) pool_free(d_tab);
                return cuda_error(e, "accept table upload");
            }
            q->tables.emplace(acc, d_tab);
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
    const size_t smem = rle_smem_bytes();
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
        e = cudaFuncSetAttribute(rle_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) rle_count_kernel<<<q->ntiles, kStagedThreads, smem, s>>>(a);
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
