// K3/K4: threshold and symmetric queries over EWAH-style run-length-encoded
// bitmaps, decoded on the device (sm_100a).
//
// Stream format (reference bitmaps.py:27-40): a marker word
//   bit 0 = fill bit, bits 1-32 = fill run (words), bits 33-63 = literal count
// followed by that many literal ("dirty") words; coverage shorter than
// ceil(r/64) words is an implicit zero tail (bitmaps.py:215-219).
//
// K3 rle_directory_kernel -- one warp per stream walks the marker chain once
//   (inputs are immutable, so the result is cached in the query object).  A
//   32-word window is loaded coalesced; the chain inside it is followed with
//   warp shuffles, marker lanes are flagged with a ballot, their word
//   positions come from a warp prefix sum, and every tile boundary a marker's
//   run covers is recorded as a directory entry (marker index, run start).
//   Dirty runs longer than the window are skipped without being loaded.
//   Malformed streams (truncated literal group, coverage beyond ceil(r/64)
//   words) raise FormatError like RleBitmap.iter_word_segments (:210-217).
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
#include <string.h>

#include <algorithm>
#include <vector>

#include "bq_internal.h"

namespace bq {

constexpr int kRleTile = 4096;        // output words per K4 tile (and directory granularity)
constexpr int kRleThreads = 256;
constexpr int kSlotsPerBatch = 256;   // undecided words resolved per phase-C pass
constexpr uint16_t kNoSlot = 0xFFFF;
constexpr int kStageWords = 4096;       // words per cp.async stage buffer (two buffers)
constexpr int kMaxStagedInputs = 4096;  // N up to this stages segments through shared memory
constexpr int kMaxBatches = 64;
constexpr size_t kCntBytes = (size_t)(kRleTile + 4) * 4;
constexpr size_t kPhaseCBytes = (size_t)kSlotsPerBatch * 128 + (size_t)kRleTile * 4 + (size_t)kSlotsPerBatch * 2;
constexpr size_t kRegionBytes = (2 * (size_t)kStageWords * 8 > kPhaseCBytes) ? 2 * (size_t)kStageWords * 8 : kPhaseCBytes;

inline size_t rle_smem_bytes(bool staged, int n) {
    return kCntBytes + kRegionBytes + (staged ? (((size_t)n + 1) * 4 + 15) / 16 * 16 : 0);
}

enum { RLE_ERR_TRUNCATED = 1, RLE_ERR_OVERLONG = 2, RLE_ERR_BEYOND_R = 3 };

struct RleDirArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    int n;
    uint64_t total_words;  // ceil(r/64)
    uint64_t tail_mask;    // valid bits of the last word when r % 64 != 0, else 0
    uint32_t ntiles;
    uint2 *dir;            // [n][ntiles]: (marker index, run start word)
    int *err;              // first error code
    unsigned long long *err_stream;
};

__device__ __forceinline__ void rle_fail(const RleDirArgs &a, int code, int stream) {
    if (atomicCAS(a.err, 0, code) == 0) atomicExch(a.err_stream, (unsigned long long)stream);
}

__global__ void __launch_bounds__(128) rle_directory_kernel(const __grid_constant__ RleDirArgs a) {
    const int lane = threadIdx.x & 31;
    const int stream = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (stream >= a.n) return;
    const uint64_t *s = a.ptrs[stream];
    const uint64_t L = a.lens[stream];
    uint2 *dir = a.dir + (size_t)stream * a.ntiles;
    uint64_t i = 0;     // stream index of the next marker
    uint64_t pos = 0;   // word position where that marker's fill run starts
    while (i < L) {
        const uint64_t idx = i + lane;
        const uint64_t w = idx < L ? __ldg(s + idx) : 0ull;
        const uint64_t run = (w >> 1) & 0xFFFFFFFFull;
        const uint64_t dirty = w >> 33;
        const uint64_t nxt = (uint64_t)lane + 1 + dirty;
        // follow the chain from lane 0 (a marker) through the window
        uint32_t mask = 0;
        uint64_t cur = 0;
        while (cur < 32 && i + cur < L) {
            mask |= 1u << cur;
            cur = __shfl_sync(0xffffffffu, nxt, (int)cur);
        }
        const bool is_m = (mask >> lane) & 1u;
        const uint64_t span = is_m ? run + dirty : 0ull;
        // exclusive prefix sum of spans over marker lanes
        uint64_t incl = span;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint64_t start = pos + incl - span;
        const uint64_t end = start + span;
        if (is_m) {
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
            // record every tile boundary b with start <= b < end
            uint64_t b = (start + kRleTile - 1) / kRleTile * kRleTile;
            for (; b < end && b < a.total_words; b += kRleTile)
                dir[b / kRleTile] = make_uint2((uint32_t)idx, (uint32_t)start);
        }
        const uint64_t total = __shfl_sync(0xffffffffu, incl, 31);
        pos += total;
        i += cur;
        if (*((volatile int *)a.err)) break;
    }
    // tiles past the encoded coverage: stream exhausted, implicit zero tail
    uint64_t b = (pos + kRleTile - 1) / kRleTile * kRleTile;
    for (uint64_t t = b / kRleTile + lane; t < a.ntiles; t += 32) dir[t] = make_uint2((uint32_t)L, (uint32_t)pos);
}

struct RleCountArgs {
    const uint64_t *const *ptrs;
    const uint64_t *lens;
    const uint2 *dir;
    int n;
    uint64_t total_words;
    uint32_t ntiles;
    uint64_t last_mask;
    const uint32_t *accept_bits;  // (n + 1) bits
    const uint32_t *const_until;  // [n + 1]: largest j >= k with accept[k..j] constant
    uint64_t *out;
    unsigned long long *popcnt;
};

__device__ __forceinline__ bool accept_at(const uint32_t *bits, uint32_t c) { return (bits[c >> 5] >> (c & 31)) & 1u; }

// Walk stream `st` across tile [ts, te) from its directory entry; Visit(fs, fe, bit, ds, de, lit)
// is called for each marker whose runs intersect the tile (fill [fs,fe), dirty [ds,de) with the
// first literal at stream index lit).
template <typename Visit>
__device__ __forceinline__ void walk_tile(const RleCountArgs &a, int st, uint32_t tile, uint64_t ts, uint64_t te,
                                          Visit &&visit) {
    const uint64_t *s = a.ptrs[st];
    const uint64_t L = a.lens[st];
    const uint2 e = a.dir[(size_t)st * a.ntiles + tile];
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

__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Exclusive prefix sum of arr[0..n) in place (arr[n] receives the total).
__device__ void block_exclusive_scan(uint32_t *arr, int n, uint32_t *warp_sums) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + kRleThreads - 1) / kRleThreads;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    uint32_t sum = 0;
    for (int k = lo; k < hi; ++k) sum += arr[k];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    uint32_t off = incl - sum;
    for (int w = 0; w < warp; ++w) off += warp_sums[w];
    for (int k = lo; k < hi; ++k) {
        const uint32_t v = arr[k];
        arr[k] = off;
        off += v;
    }
    if (tid == kRleThreads - 1) arr[n] = off;
    __syncthreads();
}

// Marker sweep of one stream over tile [ts, te) reading words from `src` (shared
// memory or global), src[0] being the stream's marker at directory index e.x.
template <typename Visit>
__device__ __forceinline__ void walk_words(const uint64_t *src, uint64_t first, uint64_t L, uint64_t pos,
                                           uint64_t ts, uint64_t te, Visit &&visit) {
    uint64_t i = first;
    while (i < L && pos < te) {
        const uint64_t mk = src[i - first];
        const uint64_t run = (mk >> 1) & 0xFFFFFFFFull;
        const uint64_t dirty = mk >> 33;
        const uint64_t fe = pos + run, de = fe + dirty;
        if (de > ts) visit(pos, fe, (uint32_t)(mk & 1), fe, de);
        pos = de;
        i += 1 + dirty;
    }
}

// STAGED: the tile's segment of every stream (from its directory entry to the
// marker covering the next tile boundary) is copied to shared memory with
// cp.async in batches of kStageWords words, double buffered, so the
// pointer-chasing marker walk reads shared memory while the next batch streams
// in from HBM at full width.  Without staging (N > kMaxStagedInputs) the walk
// reads global memory directly.
template <bool STAGED>
__global__ void __launch_bounds__(kRleThreads, 2) rle_count_kernel(const __grid_constant__ RleCountArgs a) {
    extern __shared__ __align__(16) uint8_t rle_smem[];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rle_smem);  // [kRleTile + 4] packed (ones | dirty << 16)
    uint8_t *region = rle_smem + kCntBytes;                  // phase A: stage buffers; phase C: bit counters
    uint64_t *stage = reinterpret_cast<uint64_t *>(region);  // [2][kStageWords]
    uint32_t (*bitcnt)[32] = reinterpret_cast<uint32_t (*)[32]>(region);                   // [kSlotsPerBatch][32]
    uint16_t *slot_of = reinterpret_cast<uint16_t *>(region + kSlotsPerBatch * 128);       // [kRleTile]
    uint16_t *undecided = slot_of + kRleTile;                                                // [kRleTile]
    uint16_t *slot_word = undecided + kRleTile;                                              // [kSlotsPerBatch]
    uint32_t *seg_off = reinterpret_cast<uint32_t *>(rle_smem + kCntBytes + kRegionBytes);  // [n + 1] (STAGED)
    __shared__ uint32_t n_undecided;
    __shared__ uint32_t warp_sums[kRleThreads / 32];
    __shared__ uint32_t bounds[kMaxBatches + 1];
    __shared__ uint32_t n_batches;

    const uint32_t tile = blockIdx.x;
    const uint64_t ts = (uint64_t)tile * kRleTile;
    const uint64_t te = min(ts + (uint64_t)kRleTile, a.total_words);
    const int width = (int)(te - ts);
    const int tid = threadIdx.x;
    const int n = a.n;

    for (int k = tid; k <= kRleTile; k += kRleThreads) cnt[k] = 0u;
    if (tid == 0) n_undecided = 0;

    auto sweep = [&](uint64_t fs, uint64_t fe, uint32_t bit, uint64_t ds, uint64_t de) {
        if (bit && fe > ts && fs < te) {
            atomicAdd(&cnt[max(fs, ts) - ts], 1u);
            atomicAdd(&cnt[min(fe, te) - ts], 0xFFFFFFFFu);
        }
        if (de > ds && de > ts && ds < te) {
            atomicAdd(&cnt[max(ds, ts) - ts], 0x10000u);
            atomicAdd(&cnt[min(de, te) - ts], 0xFFFF0000u);
        }
    };

    // ---- A: run sweep over markers only -> difference array ------------------
    if constexpr (!STAGED) {
        __syncthreads();
        for (int st = tid; st < n; st += kRleThreads) {
            const uint2 e = a.dir[(size_t)st * a.ntiles + tile];
            const uint64_t *s = a.ptrs[st];
            walk_words(s + e.x, e.x, a.lens[st], e.y, ts, te, sweep);
        }
    } else {
        // segment length of every stream in this tile, then offsets
        for (int st = tid; st < n; st += kRleThreads) {
            const uint64_t L = a.lens[st];
            const uint32_t first = a.dir[(size_t)st * a.ntiles + tile].x;
            const uint64_t next = (tile + 1 < a.ntiles) ? a.dir[(size_t)st * a.ntiles + tile + 1].x : L;
            const uint64_t end = min(next + 1, L);
            seg_off[st] = (first < L) ? (uint32_t)(end - first) : 0u;
        }
        __syncthreads();
        block_exclusive_scan(seg_off, n, warp_sums);
        int s_done = 0;
        while (s_done < n) {
            if (tid == 0) {  // greedy batches of consecutive streams that fit one stage buffer
                uint32_t nb = 0;
                int s = s_done;
                bounds[0] = (uint32_t)s;
                while (s < n && nb < kMaxBatches) {
                    int lo = s + 1, hi = n;  // largest s1 in [s+1, n] with seg_off[s1] - seg_off[s] <= kStageWords
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (seg_off[mid] - seg_off[s] <= (uint32_t)kStageWords) lo = mid;
                        else hi = mid - 1;
                    }
                    s = lo;
                    bounds[++nb] = (uint32_t)s;
                }
                n_batches = nb;
            }
            __syncthreads();
            const uint32_t nb = n_batches;
            auto issue = [&](uint32_t k) {
                const int s0 = (int)bounds[k], s1 = (int)bounds[k + 1];
                if (seg_off[s1] - seg_off[s0] > (uint32_t)kStageWords) return;  // one oversize stream: walk from HBM
                uint64_t *buf = stage + (size_t)(k & 1) * kStageWords;
                const int lane = tid & 31;
                for (int st = s0 + (tid >> 5); st < s1; st += kRleThreads / 32) {
                    const uint32_t len = seg_off[st + 1] - seg_off[st];
                    if (!len) continue;
                    const uint64_t *src = a.ptrs[st] + a.dir[(size_t)st * a.ntiles + tile].x;
                    uint64_t *dst = buf + (seg_off[st] - seg_off[s0]);
                    for (uint32_t j = lane; j < len; j += 32) cp_async8(dst + j, src + j);
                }
            };
            issue(0);
            cp_async_commit();
            for (uint32_t k = 0; k < nb; ++k) {
                if (k + 1 < nb) {
                    issue(k + 1);
                    cp_async_commit();
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const int s0 = (int)bounds[k], s1 = (int)bounds[k + 1];
                const bool oversize = seg_off[s1] - seg_off[s0] > (uint32_t)kStageWords;
                const uint64_t *buf = stage + (size_t)(k & 1) * kStageWords;
                for (int st = s0 + tid; st < s1; st += kRleThreads) {
                    const uint2 e = a.dir[(size_t)st * a.ntiles + tile];
                    const uint64_t *src = oversize ? a.ptrs[st] + e.x : buf + (seg_off[st] - seg_off[s0]);
                    walk_words(src, e.x, a.lens[st], e.y, ts, te, sweep);
                }
                __syncthreads();
            }
            s_done = (int)bounds[nb];
        }
    }
    __syncthreads();

    // ---- inclusive prefix scan of cnt[0..kRleTile) (16 words per thread) ------
    constexpr int kPer = kRleTile / kRleThreads;
    uint32_t local[kPer];
    uint32_t run_sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        run_sum += cnt[tid * kPer + k];
        local[k] = run_sum;
    }
    uint32_t incl = run_sum;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    uint32_t warp_off = 0;
    for (int w = 0; w < warp; ++w) warp_off += warp_sums[w];
    const uint32_t excl = warp_off + incl - run_sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) cnt[tid * kPer + k] = local[k] + excl;
    for (int k = tid; k < kRleTile; k += kRleThreads) slot_of[k] = kNoSlot;
    __syncthreads();

    // ---- B: decide from (k, d) ----------------------------------------------
    unsigned long long pc = 0;
    for (int k = tid; k < width; k += kRleThreads) {
        const uint32_t c = cnt[k];
        const uint32_t ones = c & 0xFFFFu, dirty = c >> 16;
        if (ones + dirty <= __ldg(a.const_until + ones)) {
            uint64_t w = accept_at(a.accept_bits, ones) ? ~0ull : 0ull;
            if (ts + k == a.total_words - 1) w &= a.last_mask;
            a.out[ts + k] = w;
            pc += __popcll(w);
        } else {
            undecided[atomicAdd(&n_undecided, 1u)] = (uint16_t)k;
        }
    }
    __syncthreads();
    const uint32_t nu = n_undecided;

    // ---- C: read dirty literals only where the fills leave the outcome open ----
    for (uint32_t base = 0; base < nu; base += kSlotsPerBatch) {
        const uint32_t nb = min((uint32_t)kSlotsPerBatch, nu - base);
        for (uint32_t u = tid; u < nb; u += kRleThreads) {
            const uint16_t wk = undecided[base + u];
            slot_word[u] = wk;
            slot_of[wk] = (uint16_t)u;
        }
        for (int k = tid; k < kSlotsPerBatch * 32; k += kRleThreads) (&bitcnt[0][0])[k] = 0u;
        __syncthreads();
        for (int st = tid; st < a.n; st += kRleThreads) {
            walk_tile(a, st, tile, ts, te,
                      [&](uint64_t, uint64_t, uint32_t, uint64_t ds, uint64_t de, uint64_t lit, const uint64_t *s) {
                          const uint64_t lo = max(ds, ts), hi = min(de, te);
                          for (uint64_t p = lo; p < hi; ++p) {
                              const uint16_t u = slot_of[p - ts];
                              if (u == kNoSlot) continue;
                              uint64_t x = __ldg(s + lit + (p - ds));
                              while (x) {
                                  const int b = __ffsll((long long)x) - 1;
                                  atomicAdd(&bitcnt[u][b & 31], (b < 32) ? 1u : 0x10000u);
                                  x &= x - 1;
                              }
                          }
                      });
        }
        __syncthreads();
        for (uint32_t u = tid; u < nb; u += kRleThreads) {
            const uint16_t wk = slot_word[u];
            const uint32_t ones = cnt[wk] & 0xFFFFu;
            uint64_t w = 0;
            for (int b = 0; b < 64; ++b) {
                const uint32_t cb = (bitcnt[u][b & 31] >> ((b >> 5) * 16)) & 0xFFFFu;
                if (accept_at(a.accept_bits, ones + cb)) w |= 1ull << b;
            }
            if (ts + wk == a.total_words - 1) w &= a.last_mask;
            a.out[ts + wk] = w;
            pc += __popcll(w);
            slot_of[wk] = kNoSlot;
        }
        __syncthreads();
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
    uint32_t ntiles;
    void *mem;  // ptr table | len table | directory | error words
    const uint64_t **d_ptrs;
    uint64_t *d_lens;
    uint2 *d_dir;
    uint64_t dir_bytes;
};

extern "C" {

BQ_API int bq_rle_query_create(const bq_rle_span *streams, int n, uint64_t r_bits, int device, bq_rle_query **out) {
    if (!out) return set_error(BQ_EINPUT, "out is NULL");
    *out = nullptr;
    if (n < 1) return set_error(BQ_EINPUT, "need at least one input bitmap");
    if (n > BQ_MAX_INPUTS) return set_error(BQ_EINPUT, "%d inputs exceed BQ_MAX_INPUTS=%d", n, BQ_MAX_INPUTS);
    if (!streams) return set_error(BQ_EINPUT, "streams is NULL");
    const uint64_t total = word_count(r_bits);
    if (total >= (1ull << 32)) return set_error(BQ_EINPUT, "bit_length too large for the RLE directory (< 2^38 bits)");
    for (int i = 0; i < n; ++i) {
        if (streams[i].n_words >= (1ull << 32))
            return set_error(BQ_EINPUT, "stream %d longer than 2^32 words", i);
        if (streams[i].n_words && !streams[i].words) return set_error(BQ_EINPUT, "stream %d is NULL", i);
        if (reinterpret_cast<uintptr_t>(streams[i].words) & 7)
            return set_error(BQ_EINPUT, "stream %d: device words must be 8-byte aligned", i);
    }
    int rc = use_device(device);
    if (rc) return rc;
    const uint32_t ntiles = (uint32_t)((total + kRleTile - 1) / kRleTile);
    const size_t tab = (size_t)n * 16;
    const size_t dirb = (size_t)n * ntiles * sizeof(uint2);
    const size_t bytes = tab + dirb + 64;
    bq_rle_query *q = new bq_rle_query();
    q->device = device;
    q->n = n;
    q->r_bits = r_bits;
    q->total_words = total;
    q->ntiles = ntiles;
    q->dir_bytes = dirb;
    cudaError_t e = cudaMalloc(&q->mem, bytes);
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
        cudaFree(q->mem);
        delete q;
        return cuda_error(e, "rle query setup");
    }
    if (ntiles) {
        RleDirArgs a;
        a.ptrs = q->d_ptrs;
        a.lens = q->d_lens;
        a.n = n;
        a.total_words = total;
        a.tail_mask = (r_bits % W) ? ((1ull << (r_bits % W)) - 1) : 0ull;
        a.ntiles = ntiles;
        a.dir = q->d_dir;
        a.err = d_err;
        a.err_stream = d_err_stream;
        const int warps_per_block = 4;
        rle_directory_kernel<<<(n + warps_per_block - 1) / warps_per_block, 32 * warps_per_block>>>(a);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        int herr[4] = {0, 0, 0, 0};
        if (e == cudaSuccess) e = cudaMemcpy(herr, d_err, 16, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            cudaFree(q->mem);
            delete q;
            return cuda_error(e, "rle_directory_kernel");
        }
        if (herr[0]) {
            unsigned long long bad = (unsigned long long)(uint32_t)herr[2] | ((unsigned long long)(uint32_t)herr[3] << 32);
            cudaFree(q->mem);
            delete q;
            if (herr[0] == RLE_ERR_TRUNCATED)
                return set_error(BQ_EFORMAT, "stream %llu: marker announces more literal words than present", bad);
            if (herr[0] == RLE_ERR_BEYOND_R)
                return set_error(BQ_EFORMAT, "stream %llu: set bits at positions >= bit_length", bad);
            return set_error(BQ_EFORMAT, "stream %llu: encoded words exceed bit_length", bad);
        }
    }
    *out = q;
    return BQ_OK;
}

BQ_API void bq_rle_query_destroy(bq_rle_query *q) {
    if (!q) return;
    if (q->device >= 0) cudaSetDevice(q->device);
    cudaFree(q->mem);
    delete q;
}

BQ_API uint64_t bq_rle_query_directory_bytes(const bq_rle_query *q) { return q ? q->dir_bytes : 0; }

static int rle_eval(bq_rle_query *q, const std::vector<uint8_t> &acc, uint64_t *d_out, unsigned long long *d_popcnt,
                    void *stream) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    if (q->total_words && !d_out) return set_error(BQ_EINPUT, "d_out is NULL");
    int rc = use_device(q->device);
    if (rc) return rc;
    if (!q->total_words) return BQ_OK;
    const int n = q->n;
    // accept bits and const_until table (host, O(n))
    const size_t nbits_words = (size_t)(n + 1 + 31) / 32;
    std::vector<uint32_t> host(nbits_words + (size_t)n + 1, 0u);
    for (int k = 0; k <= n; ++k)
        if (acc[k]) host[k >> 5] |= 1u << (k & 31);
    uint32_t *cu = host.data() + nbits_words;
    cu[n] = (uint32_t)n;
    for (int k = n - 1; k >= 0; --k) cu[k] = (acc[k] == acc[k + 1]) ? cu[k + 1] : (uint32_t)k;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void *d_tab = nullptr;
    const size_t bytes = host.size() * 4;
    cudaError_t e = cudaMallocAsync(&d_tab, bytes, s);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(accept)");
    e = cudaMemcpyAsync(d_tab, host.data(), bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync(accept)");
    RleCountArgs a;
    a.ptrs = q->d_ptrs;
    a.lens = q->d_lens;
    a.dir = q->d_dir;
    a.n = n;
    a.total_words = q->total_words;
    a.ntiles = q->ntiles;
    a.last_mask = (q->r_bits % W) ? ((1ull << (q->r_bits % W)) - 1) : ~0ull;
    a.accept_bits = static_cast<const uint32_t *>(d_tab);
    a.const_until = static_cast<const uint32_t *>(d_tab) + nbits_words;
    a.out = d_out;
    a.popcnt = d_popcnt;
    const bool staged = n <= kMaxStagedInputs;
    const size_t smem = rle_smem_bytes(staged, n);
    if (staged) {
        e = cudaFuncSetAttribute(rle_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) rle_count_kernel<true><<<q->ntiles, kRleThreads, smem, s>>>(a);
    } else {
        e = cudaFuncSetAttribute(rle_count_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) rle_count_kernel<false><<<q->ntiles, kRleThreads, smem, s>>>(a);
    }
    if (e != cudaSuccess) {
        cudaFreeAsync(d_tab, s);
        return cuda_error(e, "cudaFuncSetAttribute(rle_count_kernel)");
    }
    e = cudaGetLastError();
    cudaFreeAsync(d_tab, s);
    if (e != cudaSuccess) return cuda_error(e, "rle_count_kernel launch");
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
