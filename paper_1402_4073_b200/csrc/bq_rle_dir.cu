// K3: the tile directory of n RLE streams in one streaming pass (sm_100a).
//
// The directory row of tile boundary b for a stream is the marker whose runs
// cover word b: (its stream index, the word where its fill starts).  Finding it
// means following the stream's marker chain (bitmaps.py:196-219) -- a marker is
// only recognisable from the previous one -- so a plain walk is one dependent
// step per marker, ~142k per C4 stream.  This kernel cuts every stream into
// segments of kSegWords stream words and walks all segments at once:
//
//  * Speculative entry.  A segment's chain enters at the first marker at or
//    after its first word.  One lane per segment guesses it from the kHalo words
//    before the segment: each of those words is taken as a marker in turn, its
//    chain followed to the first position >= the segment start, and the position
//    most of the eight chains land on (the smallest on a tie) is the guess.  True
//    markers all land on the true entry, and literal words taken as markers
//    mostly fall through to it (a literal with a zero dirty field steps to the next
//    word).  On C4 streams the guess was right for every segment measured.
//  * Walk.  From its entry, the lane walks its segment in shared memory (the
//    CTA's block of 32 segments is staged by one TMA bulk copy), summing the words
//    the markers cover; its exit is the first chain position past the segment.
//  * Resolution.  A segment's guess is right iff it equals the previous
//    segment's exit (or, if that exit lies past the segment, the segment holds no
//    marker start at all).  Within a block this is checked lane by lane; across
//    blocks by a decoupled look-back: blocks take tickets in (block, stream)
//    order, each publishes its exit and end position as soon as its own entry is
//    known, and the next block of the stream spins on that word.  A wrong guess
//    is repaired by re-walking that segment from the true entry (shared memory,
//    no second HBM read), so the result is exact whatever the guesses.
//  * Directory.  With its true entry and absolute word position, every lane
//    walks its segment once more from shared memory and writes the row of every
//    tile boundary its markers cover.  Validation is iter_word_segments' /
//    decompress's: a chain leaving the stream early is a truncated literal group,
//    coverage past ceil(r/64) words is overlong, set bits >= r are beyond r
//    (bitmaps.py:210-217, :428-431), in that order of precedence.
//
// HBM traffic is one read of the streams plus the directory (8 bytes per tile
// and stream); the old form (one warp per stream following the chain window by
// window, then a second pass over all windows) read the streams twice and was
// latency-bound on the serial chain.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "bq_internal.h"

namespace bq {

#ifndef BQ_DIR_SEG
#define BQ_DIR_SEG 32
#endif
// Measurement probe (never in the shipped library; profiles/README.md): the second walk also
// issues phase A's difference-array updates as global reductions into one array for the whole
// word range, the cost a single-read fresh query would add to this kernel.
#ifndef BQ_K3_RED_PROBE
#define BQ_K3_RED_PROBE 0
#endif
#ifndef BQ_DIR_LDS
#define BQ_DIR_LDS 1
#endif

constexpr int kSegWords = BQ_DIR_SEG;                // stream words per segment (one lane)
constexpr int kBlockWords = kSegWords * 32;          // one warp = one block of 32 segments
constexpr int kHalo = 8;                             // words before a segment holding its entry guesses
// Staging: a group of kGroup consecutive segments is copied by one TMA bulk copy
// into one slot (its lanes' words are contiguous there; the halo words of a lane are
// the end of its left neighbour's segment, in the same slot or the previous one, and
// lane 0's come from HBM); slot stride = 16 bytes mod 128 so consecutive slots start
// in different shared-memory banks.  32-word segments in groups of 4: 130-word slots,
// 8.3 KB per warp, 27 warps per SM.  C4 directory: 64-word segments with per-lane
// slots holding their own halo 0.90 ms; per-lane slots without the halo 0.80;
// 48-word per-lane 0.77; 48-word groups of 2 / 4 / 8 0.735 / 0.721 / 0.733;
// 32-word groups of 2 / 4 / 8 0.748 / 0.687 / 0.711; 24-word groups of 4 0.85.
#ifndef BQ_DIR_GROUP
#define BQ_DIR_GROUP 4
#endif
constexpr int kGroup = BQ_DIR_GROUP;  // consecutive segments staged by one bulk copy into one slot
constexpr int kSlotWords = ((kGroup * kSegWords + 15) / 16) * 16 + 2;

struct DirArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    int n;
    uint64_t n_recip;            // ceil(2^64 / n), 0 when n = 1
    uint64_t total_words;        // ceil(r / 64)
    uint64_t tail_mask;          // valid bits of word total_words - 1 when r % 64 != 0, else 0
    uint32_t tile0, nrows;       // directory rows: tile boundaries tile0 .. tile0 + nrows - 1
    uint2 *dir;                  // [nrows][n] (marker index, fill start word)
    uint32_t full_levels;        // tickets < full_levels * n: block t / n of stream t % n (every stream has them)
    const uint2 *jobs;           // later tickets: (stream, block), block-major
    const uint32_t *nblocks;     // per stream
    unsigned long long *link;    // [block][stream]: exit | end position << 32, ~0 until published
    unsigned int *ticket;
    unsigned long long *err;     // min over (stream << 32 | precedence): the first failing stream
#if BQ_K3_RED_PROBE
    uint32_t *probe;             // measurement only: packed difference array of the whole range
#endif
};

enum { DIR_ERR_TRUNCATED = 0, DIR_ERR_OVERLONG = 1, DIR_ERR_BEYOND_R = 2 };

__device__ __forceinline__ void dir_fail(const DirArgs &a, uint32_t code, uint32_t stream) {
    atomicMin(a.err, ((unsigned long long)stream << 32) | code);
}

// The link word is self-contained (exit and end position in one 64-bit store), and
// nothing else the consumer reads depends on the producer: relaxed accesses at gpu
// scope suffice (no fence on the producer's critical path).
__device__ __forceinline__ unsigned long long ld_link(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_link(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

__global__ void __launch_bounds__(32) rle_dir_kernel(const __grid_constant__ DirArgs a) {
    __shared__ __align__(16) uint64_t slots[(32 / kGroup) * kSlotWords];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x;

    unsigned int t = 0;
    // tickets in start order: a block's predecessor started earlier.  The counter starts at
    // 0xFFFFFFFF (it shares one 0xFF memset with the links and the error word).  A ticket
    // taken any earlier than its block starts (persistent warps prefetching the next one,
    // even after publishing: 0.78 / 0.70 ms instead of 0.66 on C4) lets start order drift from
    // ticket order, and blocks then spin on predecessors whose warps are still busy.
    if (lane == 0) t = atomicAdd(a.ticket, 1u) + 1u;
    t = __shfl_sync(0xffffffffu, t, 0);
    const uint32_t full = a.full_levels * (uint32_t)a.n;
    // t / n by a multiply with ceil(2^64 / n) (exact for t < 2^32; the host passes 0 for n = 1)
    const uint32_t tq = a.n_recip ? (uint32_t)__umul64hi((uint64_t)t, a.n_recip) : t;
    const uint2 job = t < full ? make_uint2(t - tq * (uint32_t)a.n, tq) : a.jobs[t - full];
    const uint32_t stream = job.x, blk = job.y;
    const uint64_t *s = a.ptrs[stream];
    const uint32_t L = (uint32_t)a.lens[stream];  // < 2^32 - 2 (bq_rle_query_create)
    const bool last_block = blk + 1 == a.nblocks[stream];  // loaded here: the publish below is on the look-back chain
    const uint64_t total = a.total_words;

    // ---- this lane's segment [q, qe) and its staging: words [q - kHalo, qe) --------
    const uint32_t q = blk * (uint32_t)kBlockWords + (uint32_t)lane * kSegWords;
    const bool active = q < L;
    const uint32_t qe = active ? min(q + (uint32_t)kSegWords, L) : q;
    // the lane's group of kGroup segments [gq, gqe), copied by its first lane
    const uint32_t gq = blk * (uint32_t)kBlockWords + (uint32_t)(lane / kGroup) * (kGroup * kSegWords);
    const uint32_t gqe = gq < L ? min(gq + (uint32_t)(kGroup * kSegWords), L) : gq;
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(s + gq) & ~(uintptr_t)15;
    const uintptr_t g1 = (reinterpret_cast<uintptr_t>(s + gqe) + 15) & ~(uintptr_t)15;
    const uint32_t bytes = (lane % kGroup == 0 && gq < L) ? (uint32_t)(g1 - g0) : 0u;
    uint64_t *slot = slots + (lane / kGroup) * kSlotWords;
    // stream word p is slot[p - sbase] (sbase = q or q - 1 after the widening: -1 at a
    // segment that starts 8 bytes into a 16-byte line)
    const int64_t sbase = ((intptr_t)g0 - reinterpret_cast<intptr_t>(s)) / 8;
    // the walks load through 32-bit shared addresses (no generic-to-shared conversion per step)
    const uint32_t slot_s = (uint32_t)__cvta_generic_to_shared(slot);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_s), "r"(32) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (bytes) {
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar_s),
                     "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(slot)),
                     "l"(g0), "r"(bytes), "r"(bar_s)
                     : "memory");
    } else {
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar_s) : "memory");
    }
    // lane 0's halo words are the previous block's last words, read from HBM: issued here so
    // their latency hides behind the copies (after the wait they stalled the whole warp)
    uint64_t halo0[kHalo];
#pragma unroll
    for (int j = 0; j < kHalo; ++j) halo0[j] = (lane == 0 && active && q > 0) ? __ldg(s + (q - kHalo + j)) : 0ull;
    // the previous block's exit is published by now in the common case: fetch it while
    // the copies land
    uint64_t link_prev = 0;
    if (blk > 0 && lane == 0) link_prev = ld_link(a.link + (size_t)(blk - 1) * a.n + stream);
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(done)
                         : "r"(bar_s)
                         : "memory");
    }

    // speculative entry: the landing most of the kHalo hypotheses reach (smallest on a tie)
    uint32_t entry = q;
    // the halo words [q - kHalo, q): the end of the left neighbour's slot (its sbase by shuffle;
    // it is active whenever this lane is), lane 0 reads the previous block's last words
    const int64_t sbase_left = __shfl_up_sync(0xffffffffu, sbase, 1);
    const uint32_t slot_left = __shfl_up_sync(0xffffffffu, slot_s, 1);
    const uint32_t halo_s = lane ? slot_left + (uint32_t)((int64_t)q - kHalo - sbase_left) * 8u : 0u;
    if (active && q > 0) {
        // landings saturate at 2^32 - 1 (beyond any stream): never a valid entry.  A
        // hypothesis whose next marker is a later halo word shares that word's root (the
        // halo word whose chain leaves the halo); each root gets the votes of the
        // hypotheses on it, kept as 4-bit counters in one word (no per-pair comparisons)
        static_assert(kHalo <= 8, "4-bit root indices and vote counters");
        uint32_t nxs[kHalo];
        uint32_t rootp = 0, votes = 0;
#pragma unroll
        for (int j = kHalo - 1; j >= 0; --j) {
            const uint32_t h = q - kHalo + j;
            const uint64_t hw = lane ? lds64(halo_s + (uint32_t)j * 8u) : halo0[j];
            // h + 1 + dirty, saturated: dirty < 2^31 and h + 1 < 2^32, so a wrapped sum is < dirty
            const uint32_t hd = (uint32_t)(hw >> 33);
            const uint32_t hsum = h + 1u + hd;
            const uint32_t nx = hsum < hd ? 0xFFFFFFFFu : hsum;
            nxs[j] = nx;
            // nx > h, so a landing inside the halo is a later halo word k > j
            const uint32_t r = nx < q ? (rootp >> (4u * (nx - (q - kHalo)))) & 15u : (uint32_t)j;
            rootp |= r << (4 * j);
            votes += 1u << (4u * r);
        }
        uint32_t best = 0, pick = 0xFFFFFFFFu;
#pragma unroll
        for (int r = 0; r < kHalo; ++r) {
            const uint32_t c = (votes >> (4 * r)) & 15u;
            if (c > best || (c == best && c && nxs[r] < pick)) {
                best = c;
                pick = nxs[r];
            }
        }
        entry = min(pick, L + 1);
    }
    // walk from slot index i to the first chain position >= qe, summing the words the
    // markers cover (i stays < 2^32: it is < qe - sbase before a step, dirty < 2^31)
    const uint32_t iend = (uint32_t)((int64_t)qe - sbase);
    auto walk = [&](uint32_t from, uint64_t &span) -> uint64_t {
        span = 0;
        uint32_t i = (uint32_t)((int64_t)from - sbase);
        while (i < iend) {
            const uint64_t w = BQ_DIR_LDS ? lds64(slot_s + i * 8u) : slot[i];
            const uint32_t dirty = (uint32_t)(w >> 33);
            span += (uint64_t)(uint32_t)(w >> 1) + dirty;
            i += 1 + dirty;
        }
        return (uint64_t)((int64_t)i + sbase);
    };
    uint64_t span = 0, exit_ = entry;
    if (active && entry < qe) exit_ = walk(entry, span);

    // ---- resolution: every entry must be the previous segment's exit -------------
    // All lanes check at once; a lane whose predecessor's exit lies past its segment
    // holds no marker start (it passes the exit through), a lane whose guess differs
    // re-walks from the true entry.  Repeat while any exit changed (typically never).
    // Then the inclusive prefix of the spans (positions relative to the block).
    uint64_t incl = 0;
    auto resolve = [&](uint64_t n_in) {
        for (;;) {
            uint64_t prev = __shfl_up_sync(0xffffffffu, exit_, 1);
            if (lane == 0) prev = n_in;
            bool changed = false;
            if (!active || prev >= qe) {
                changed = exit_ != prev || span;
                entry = (uint32_t)min(prev, (uint64_t)L + 1);
                exit_ = prev;
                span = 0;
            } else if (prev != entry) {
                entry = (uint32_t)prev;
                exit_ = walk(entry, span);
                changed = true;
            }
            if (!__ballot_sync(0xffffffffu, changed)) break;
        }
        incl = span;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
    };
    // The block resolves itself before its entry is known, on lane 0's guess: the look-back
    // chain (one hop per block of a stream, ~290 on C4) then carries only a compare, an add
    // and the store below instead of the ballot round and the prefix sum.
    const uint64_t n_guess = __shfl_sync(0xffffffffu, (uint64_t)entry, 0);
    resolve(n_guess);
    // ---- the block's entry: the previous block's exit (decoupled look-back) --------
    uint64_t n_in = 0, p_in = 0;
    if (blk > 0) {
        if (lane == 0) {
            const unsigned long long *lk = a.link + (size_t)(blk - 1) * a.n + stream;
            int spins = 0;
            while (link_prev == ~0ull) {
                if (++spins > 4) __nanosleep(64);
                link_prev = ld_link(lk);
            }
            n_in = link_prev & 0xFFFFFFFFull;
            p_in = link_prev >> 32;
        }
        n_in = __shfl_sync(0xffffffffu, n_in, 0);
        p_in = __shfl_sync(0xffffffffu, p_in, 0);
    }
    if (n_in != n_guess) resolve(n_in);  // warp-uniform; rare
    // publish this block's exit for the next block of the stream (clamped: > L is a
    // truncated group, > total overlong; both below the ~0 sentinel)
    if (lane == 31 && !last_block) {
        const uint64_t ex = min(exit_, (uint64_t)L + 1), pe = min(p_in + incl, total + 1);
        st_link(a.link + (size_t)blk * a.n + stream, ex | (pe << 32));
    }
    // absolute word positions
    const uint64_t pos0 = p_in + incl - span;
    const uint64_t p_end = __shfl_sync(0xffffffffu, p_in + incl, 31);
    const uint64_t x_end = __shfl_sync(0xffffffffu, exit_, 31);
    if (lane == 31 && last_block) {
        if (x_end > L) dir_fail(a, DIR_ERR_TRUNCATED, stream);
        else if (p_end > total) dir_fail(a, DIR_ERR_OVERLONG, stream);
    }

    // ---- directory rows of the tile boundaries this segment's markers cover ------
    // nb: the next tile boundary of the query's range (~0 past it), drow its row.  A
    // marker crossing a boundary costs one store (several only for fills longer than
    // a tile), so the warp rarely diverges here.
    const uint64_t r0 = (uint64_t)a.tile0 * kRleTile;
    const uint64_t rlim = min((uint64_t)(a.tile0 + a.nrows) * kRleTile, total);
    uint64_t nb = max((pos0 + kRleTile - 1) / kRleTile * kRleTile, r0);
    uint2 *drow = a.dir + ((nb / kRleTile) - a.tile0) * (uint64_t)a.n + stream;
    if (nb >= rlim) nb = ~0ull;
    uint64_t pos = pos0;
    uint32_t i = active ? (uint32_t)((int64_t)entry - sbase) : iend;
#if BQ_K3_RED_PROBE
    uint32_t probe_carry = 0u;
#endif
    auto dir_walk = [&](auto tail_check) {
        while (i < iend) {
            const uint64_t w = BQ_DIR_LDS ? lds64(slot_s + i * 8u) : slot[i];
            const uint32_t dirty = (uint32_t)(w >> 33);
            const uint64_t end = pos + (uint32_t)(w >> 1) + dirty;
            if (end > nb) {  // the marker covers boundary nb (< rlim)
                const uint2 v = make_uint2((uint32_t)((int64_t)i + sbase), (uint32_t)pos);
                *drow = v;
                drow += a.n;
                nb += kRleTile;
                if (end > nb || nb >= rlim) {  // rare: a fill longer than a tile, or the range's end
                    for (; end > nb && nb < rlim; nb += kRleTile, drow += a.n) *drow = v;
                    if (nb >= rlim) nb = ~0ull;
                }
            }
#if BQ_K3_RED_PROBE
            {
                const uint32_t ones = (uint32_t)w & 1u, litv = dirty ? 0x10000u : 0u;
                const uint32_t at_pos = probe_carry + ones, at_fe = litv - ones;
                if (at_pos) atomicAdd(a.probe + pos, at_pos);
                if (at_fe) atomicAdd(a.probe + pos + (uint32_t)(w >> 1), at_fe);
                probe_carry = 0u - litv;
            }
#endif
            tail_check(w, dirty, end);
            pos = end;
            i += 1 + dirty;
        }
#if BQ_K3_RED_PROBE
        if (probe_carry) atomicAdd(a.probe + pos, probe_carry);
#endif
    };
    if (a.tail_mask) {
        dir_walk([&](uint64_t w, uint32_t dirty, uint64_t end) {
            // bits >= r in the last word (bitmaps.py:70-72 via decompress :428-431)
            if (end == total && end > pos) {
                const uint64_t p = (uint64_t)((int64_t)i + sbase);
                if (dirty == 0) {
                    if (w & 1) dir_fail(a, DIR_ERR_BEYOND_R, stream);
                } else if (p + dirty < L && (__ldg(s + p + dirty) & ~a.tail_mask)) {
                    dir_fail(a, DIR_ERR_BEYOND_R, stream);
                }
            }
        });
    } else {
        dir_walk([](uint64_t, uint32_t, uint64_t) {});
    }
    // rows past the stream's coverage: exhausted stream, implicit zero tail
    if (last_block && p_end <= total) {
        const uint64_t t0 = max((p_end + kRleTile - 1) / kRleTile, (uint64_t)a.tile0);
        for (uint64_t tt = t0 + lane; tt < (uint64_t)a.tile0 + a.nrows; tt += 32)
            a.dir[(tt - a.tile0) * (uint64_t)a.n + stream] = make_uint2(L, (uint32_t)p_end);
    }
}

// Scratch of a directory build (device bytes): links, per-stream block counts, the
// job table of the partial levels, ticket and error words.
size_t rle_directory_scratch_bytes(const std::vector<uint64_t> &lens) {
    const size_t n = lens.size();
    uint64_t maxb = 1, minb = ~0ull, njobs = 0;
    for (uint64_t L : lens) {
        const uint64_t b = std::max<uint64_t>(1, (L + kBlockWords - 1) / kBlockWords);
        maxb = std::max(maxb, b);
        minb = std::min(minb, b);
        njobs += b;
    }
    if (!n) minb = 0;
    const size_t rem = njobs - minb * n;
    return ((maxb * n * 8 + 255) & ~(size_t)255) + ((n * 4 + 255) & ~(size_t)255) + ((rem * 8 + 255) & ~(size_t)255) +
           256;
}

int build_rle_directory(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const std::vector<uint64_t> &lens,
                        uint64_t total_words, uint64_t tail_mask, uint32_t tile0, uint32_t nrows, uint2 *d_dir,
                        void *d_scratch, int *err_code, uint64_t *err_stream, const void *h_extra, void *d_extra,
                        size_t extra_bytes) {
    const int n = (int)lens.size();
    *err_code = 0;
    std::vector<uint32_t> nblk(n);
    uint32_t maxb = 1, minb = ~0u;
    uint64_t njobs = 0;
    for (int i = 0; i < n; ++i) {
        nblk[i] = (uint32_t)std::max<uint64_t>(1, (lens[i] + kBlockWords - 1) / kBlockWords);
        njobs += nblk[i];
        maxb = std::max(maxb, nblk[i]);
        minb = std::min(minb, nblk[i]);
    }
    if (njobs >= (1ull << 31)) return set_error(BQ_ERESOURCE, "streams too long for one directory launch");
    // tickets block-major: block k of every stream before block k + 1 of any.  The
    // levels every stream has map arithmetically; only the rest need a table, written
    // with the block counts into a pinned staging buffer (kept between calls) so the
    // upload is one DMA; the build holds the staging lock until it has completed.
    const size_t rem = njobs - (uint64_t)minb * n;
    const size_t a_link = ((size_t)maxb * n * 8 + 255) & ~(size_t)255;
    const size_t a_nblk = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t a_jobs = (rem * 8 + 255) & ~(size_t)255;
    const size_t a_up = (a_nblk + rem * 8 + 15) & ~(size_t)15;
    const size_t up_bytes = a_up + extra_bytes;
    static std::mutex staging_mu;
    static char *staging = nullptr;
    static size_t staging_cap = 0;
    std::lock_guard<std::mutex> staging_guard(staging_mu);
    if (staging_cap < up_bytes + 16) {
        if (staging) cudaFreeHost(staging);
        staging = nullptr;
        staging_cap = 0;
        const size_t cap = std::max<size_t>(up_bytes + 16, 1 << 16);
        if (cudaHostAlloc(reinterpret_cast<void **>(&staging), cap, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            staging = nullptr;
            return set_error(BQ_ERESOURCE, "pinned staging for the directory job table");
        }
        staging_cap = cap;
    }
    memcpy(staging, nblk.data(), (size_t)n * 4);
    {
        uint2 *jt = reinterpret_cast<uint2 *>(staging + a_nblk);
        size_t k = 0;
        for (uint32_t b = minb; b < maxb; ++b)
            for (int i = 0; i < n; ++i)
                if (b < nblk[i]) jt[k++] = make_uint2((uint32_t)i, b);
    }
    // scratch: block counts | job table | links | ticket | error word (the last three are
    // adjacent: one memset)
    char *sc = static_cast<char *>(d_scratch);
    uint32_t *d_nblk = reinterpret_cast<uint32_t *>(sc);
    uint2 *d_jobs = reinterpret_cast<uint2 *>(sc + a_nblk);
    unsigned long long *d_link = reinterpret_cast<unsigned long long *>(sc + a_nblk + a_jobs);
    unsigned int *d_ticket = reinterpret_cast<unsigned int *>(sc + a_nblk + a_jobs + a_link);
    unsigned long long *d_err = reinterpret_cast<unsigned long long *>(sc + a_nblk + a_jobs + a_link + 8);
    // nblk and the job table are adjacent in both buffers: one copy
    if (extra_bytes) memcpy(staging + a_up, h_extra, extra_bytes);
    cudaError_t e = cudaMemcpyAsync(d_nblk, staging, a_nblk + rem * 8, cudaMemcpyHostToDevice, 0);
    if (e == cudaSuccess && extra_bytes)
        e = cudaMemcpyAsync(d_extra, staging + a_up, extra_bytes, cudaMemcpyHostToDevice, 0);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_link, 0xFF, a_link + 16, 0);
#if BQ_K3_RED_PROBE
    static uint32_t *probe_buf = nullptr;
    static size_t probe_cap = 0;
    const size_t probe_bytes = (total_words + 2) * 4;
    if (e == cudaSuccess && probe_cap < probe_bytes) {
        if (probe_buf) cudaFree(probe_buf);
        e = cudaMalloc(reinterpret_cast<void **>(&probe_buf), probe_bytes);
        probe_cap = e == cudaSuccess ? probe_bytes : 0;
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(probe_buf, 0, probe_bytes, 0);
#endif
    if (e == cudaSuccess) {
        DirArgs a;
        a.ptrs = d_ptrs;
        a.lens = d_lens;
        a.n = n;
        a.n_recip = n > 1 ? ~0ull / (uint64_t)n + 1 : 0ull;
        a.total_words = total_words;
        a.tail_mask = tail_mask;
        a.tile0 = tile0;
        a.nrows = nrows;
        a.dir = d_dir;
        a.full_levels = minb;
        a.jobs = d_jobs;
        a.nblocks = d_nblk;
        a.link = d_link;
        a.ticket = d_ticket;
        a.err = d_err;
#if BQ_K3_RED_PROBE
        a.probe = probe_buf;
#endif
        rle_dir_kernel<<<(unsigned)njobs, 32, 0, 0>>>(a);
        e = cudaGetLastError();
    }
    // the verdict comes back into the pinned staging buffer (a pageable destination would
    // go through the driver's own staging copy)
    unsigned long long *h_verdict = reinterpret_cast<unsigned long long *>(staging + ((up_bytes + 7) & ~(size_t)7));
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_verdict, d_err, 8, cudaMemcpyDeviceToHost, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) return cuda_error(e, "rle directory (K3)");
    const unsigned long long herr = *h_verdict;
    if (herr != ~0ull) {
        const uint32_t code = (uint32_t)(herr & 0xFFFFFFFFull);
        *err_code = code == DIR_ERR_TRUNCATED ? 1 : code == DIR_ERR_OVERLONG ? 2 : 3;
        *err_stream = herr >> 32;
    }
    return BQ_OK;
}

}  // namespace bq
