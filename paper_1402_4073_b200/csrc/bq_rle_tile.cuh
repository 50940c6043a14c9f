// Phases B and C shared by the RLE tile kernels K4 / K4c (bq_rle.cu) and K4s
// (bq_rle_sliced.cu): the whole CTA works on one 1024-word tile at a time, after
// phase A has built the tile's packed difference array cnt[0..1024] (one-fills in
// bits 0-15, dirty inputs in bits 16-31).  This is the decision half of runmerge.cdom_threshold /
// cdom_symmetric (runmerge.py:198-299): a word is decided by the fills alone when
// accept[] is constant on [ones, ones + dirty]; otherwise its
// literal bits are counted per position (dirty_segment_solver, runmerge.py:99-125).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "bq_internal.h"

namespace bq {

struct TileDecide {
    uint64_t ts;                  // first word of the tile
    int width;                    // words in the tile (1024 except the last tile)
    uint64_t total_words;
    uint64_t last_mask;           // valid bits of word total_words - 1
    const uint32_t *accept_bits;  // (n + 1) bits
    const uint32_t *const_until;  // [n + 1]: largest j >= k with accept[k..j] constant
    uint64_t *out;                // word g of the result is out[g - out_first]
    uint64_t out_first;           // first word of the query's range (a multiple of kRleTile)
    const uint32_t *breaks;       // ascending counts b where accept[b] != accept[b - 1]
    int nbreak;                   // their number, or -1 (too many: decide bit by bit)
};

// Warp inclusive prefix sum.  The shuffle's own in-range predicate guards the add
// (shfl.sync.up r|p), so no lane compare or select is spent per step.
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v, int) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
        asm("{\n\t.reg .u32 r;\n\t.reg .pred p;\n\tshfl.sync.up.b32 r|p, %0, %1, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t}\n"
            : "+r"(v)
            : "r"(o));
    return v;
}

// Inclusive prefix sum of cnt[0..kRleTile) in place; returns the tile-wide maximum
// of ones + dirty (the largest count any word of the tile can reach).
// warp_sums / warp_reach: NT / 32 words of shared memory each.
template <int NT>
__device__ __forceinline__ uint32_t tile_scan(uint32_t *cnt, uint32_t *warp_sums, uint32_t *warp_reach) {
    constexpr int kPer = kRleTile / NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t local[kPer];
    uint32_t run_sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        run_sum += cnt[tid * kPer + k];
        local[k] = run_sum;
    }
    const uint32_t incl = warp_incl_scan_u32(run_sum, lane);
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    uint32_t warp_off = 0;
    for (int w = 0; w < warp; ++w) warp_off += warp_sums[w];
    const uint32_t excl = warp_off + incl - run_sum;
    uint32_t reach = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const uint32_t c = local[k] + excl;
        cnt[tid * kPer + k] = c;
        reach = max(reach, (c & 0xFFFFu) + (c >> 16));
    }
    reach = __reduce_max_sync(0xffffffffu, reach);
    if (lane == 0) warp_reach[warp] = reach;
    __syncthreads();
    for (int w = 0; w < NT / 32; ++w) reach = max(reach, warp_reach[w]);
    return reach;
}

// Phase B: write every decided word, list the undecided ones.  Returns this
// thread's popcount share.  A tile in which no word can reach the first count
// where accept[] changes is written as constant words with 128-bit stores.
template <int NT>
__device__ __forceinline__ unsigned long long tile_decide(const TileDecide &d, const uint32_t *cnt, uint32_t reach,
                                                          uint16_t *undecided, uint32_t *n_undecided) {
    const int tid = threadIdx.x;
    unsigned long long pc = 0;
    if (reach <= __ldg(d.const_until) && d.width == kRleTile && d.ts + kRleTile < d.total_words) {
        const uint64_t w = accept_at(d.accept_bits, 0u) ? ~0ull : 0ull;
        ulonglong2 *o = reinterpret_cast<ulonglong2 *>(d.out + (d.ts - d.out_first));
        for (int k = tid; k < kRleTile / 2; k += NT) o[k] = make_ulonglong2(w, w);
        return w ? (unsigned long long)(kRleTile / NT) * 64 : 0ull;
    }
    for (int k = tid; k < d.width; k += NT) {
        const uint32_t c = cnt[k];
        const uint32_t ones = c & 0xFFFFu, dirty = c >> 16;
        if (ones + dirty <= __ldg(d.const_until + ones)) {
            uint64_t w = accept_at(d.accept_bits, ones) ? ~0ull : 0ull;
            if (d.ts + k == d.total_words - 1) w &= d.last_mask;
            d.out[d.ts - d.out_first + k] = w;
            pc += __popcll(w);
        } else {
            undecided[atomicAdd(n_undecided, 1u)] = (uint16_t)k;
        }
    }
    return pc;
}

// Phase C shared memory: slot_of[kRleTile] | slot_word[SLOTS] | soff[SLOTS + 1] |
// sfill[SLOTS] | entries[kResolveCap] (addresses of literal words, grouped by slot).
constexpr int kResolveCap = 3584;  // literal words per phase-C batch (28 KB)
template <int SLOTS, int CAP = kResolveCap>
constexpr size_t tile_resolve_bytes() {
    return (size_t)kRleTile * 2 + (size_t)SLOTS * 2 + (size_t)(SLOTS + 4) * 4 + (size_t)SLOTS * 4 + (size_t)CAP * 8;
}

template <int M>
__device__ __forceinline__ void ripple(uint64_t (&c)[16], uint64_t carry) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const uint64_t t = c[j] & carry;
        c[j] ^= carry;
        carry = t;
    }
}

// Bit-sliced sum of the n literal words at addrs[0..n) into M planes (plane j = bit j
// of the 64 counts); four independent loads in flight at a time.  The addresses are
// generic: literal words in HBM, or in the shared-memory pool K4c staged them into.
template <int M>
__device__ __forceinline__ void planes_sum(const uint64_t *addrs, uint32_t n, uint64_t (&c)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = 0ull;
    uint32_t i = 0;
    for (; i + 4 <= n; i += 4) {
        uint64_t x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = *reinterpret_cast<const uint64_t *>(addrs[i + k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) ripple<M>(c, x[k]);
    }
    for (; i < n; ++i) ripple<M>(c, *reinterpret_cast<const uint64_t *>(addrs[i]));
}

// count >= k per bit position, for the bit-sliced count c (planes 0..M-1 in use, the
// rest zero), k a runtime value
template <int M = 16>
__device__ __forceinline__ uint64_t planes_ge(const uint64_t (&c)[16], uint32_t k) {
    if (k >= (1u << M)) return 0ull;
    uint64_t gt = 0ull, eq = ~0ull;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
        const uint64_t kb = 0ull - (uint64_t)((k >> j) & 1u);
        gt |= eq & c[j] & ~kb;
        eq &= ~(c[j] ^ kb);
    }
    return gt | eq;
}

// Result word of an undecided position: accept[ones + count_b] for each bit b
// (counts in planes 0..M-1).
template <int M = 16>
__device__ __forceinline__ uint64_t decide_word(const TileDecide &d, uint32_t ones, uint32_t dirty,
                                                const uint64_t (&c)[16]) {
    if (d.nbreak >= 0) {  // accept(ones + k) = accept(ones) ^ sum over breakpoints b in (ones, ones + dirty] of [k >= b - ones]
        uint64_t w = accept_at(d.accept_bits, ones) ? ~0ull : 0ull;
        for (int i = 0; i < d.nbreak; ++i) {
            const uint32_t b = __ldg(d.breaks + i);
            if (b <= ones) continue;
            if (b > ones + dirty) break;
            w ^= planes_ge<M>(c, b - ones);
        }
        return w;
    }
    uint64_t w = 0;
    for (int bit = 0; bit < 64; ++bit) {
        uint32_t cb = 0;
#pragma unroll
        for (int j = 0; j < M; ++j) cb |= (uint32_t)((c[j] >> bit) & 1u) << j;
        if (accept_at(d.accept_bits, ones + cb)) w |= 1ull << bit;
    }
    return w;
}

// Phase C.  count_bits(slot_of, add) is called by every thread between barriers and
// must call add(slot, &word) for every literal word whose tile position p has
// slot_of[p] != kNoSlot.  Undecided words are taken in batches whose literal words
// (their dirty counts are known from phase B) fit the entries buffer; add() files
// each literal word's address under its slot (no load on the walk), and then one
// thread per slot loads them, several at a time, and sums them into
// bit-sliced counters in registers (a ripple of a few planes per word -- no
// atomics, no per-bit loop) and decides all 64 bits with bit-sliced comparisons
// against the accept vector's breakpoints.  A word with more dirty inputs than the
// buffer holds is resolved alone by atomic ripple-adds into shared planes.
template <int NT, int SLOTS, int CAP = kResolveCap, class CountBits>
__device__ __forceinline__ unsigned long long tile_resolve(const TileDecide &d, const uint32_t *cnt,
                                                           const uint16_t *undecided, uint32_t nu, uint8_t *region,
                                                           CountBits &&count_bits) {
    static_assert(SLOTS <= NT * 8, "batch selection scans SLOTS candidates with NT threads");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint16_t *slot_of = reinterpret_cast<uint16_t *>(region);
    uint16_t *slot_word = slot_of + kRleTile;
    uint32_t *soff = reinterpret_cast<uint32_t *>(slot_word + SLOTS);
    uint32_t *sfill = soff + SLOTS + 4;
    uint64_t *entries = reinterpret_cast<uint64_t *>(sfill + SLOTS);
    uint32_t *big = reinterpret_cast<uint32_t *>(entries);  // [16][2] planes of a word too big for entries
    __shared__ uint32_t batch_k, warp_tot[NT / 32];
    unsigned long long pc = 0;
    if (!nu) return 0;
    for (int k = tid; k < kRleTile; k += NT) slot_of[k] = kNoSlot;
    constexpr int kPer = (SLOTS + NT - 1) / NT;
    for (uint32_t base = 0; base < nu;) {
        // batch: the longest prefix of undecided[base ..] (<= SLOTS words) whose dirty counts fit CAP
        const uint32_t cand = min((uint32_t)SLOTS, nu - base);
        uint32_t dv[kPer], run = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t i = tid * kPer + q;
            dv[q] = i < cand ? (cnt[undecided[base + i]] >> 16) : 0u;
            run += dv[q];
        }
        const uint32_t incl = warp_incl_scan_u32(run, lane);
        if (lane == 31) warp_tot[warp] = incl;
        if (tid == 0) batch_k = 0;
        __syncthreads();
        uint32_t off = incl - run;
        for (int w = 0; w < warp; ++w) off += warp_tot[w];
        uint32_t kk = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t i = tid * kPer + q;
            if (i < cand && off + dv[q] <= (uint32_t)CAP) {
                kk = i + 1;
                soff[i] = off;
                sfill[i] = 0;
            }
            off += dv[q];
        }
        if (kk) atomicMax(&batch_k, kk);
        __syncthreads();
        const uint32_t nb = batch_k;
        if (nb == 0) {  // undecided[base] alone has more dirty inputs than the buffer holds
            const uint16_t wk = undecided[base];
            if (tid == 0) slot_of[wk] = 0;
            for (int k = tid; k < 32; k += NT) big[k] = 0u;
            __syncthreads();
            auto add_big = [&](uint16_t, const uint64_t *p) {
                const uint64_t x = *p;
                uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
#pragma unroll 1
                for (int j = 0; (lo | hi) && j < 16; ++j) {
                    if (lo) lo &= atomicXor(&big[2 * j], lo);
                    if (hi) hi &= atomicXor(&big[2 * j + 1], hi);
                }
            };
            count_bits(static_cast<const uint16_t *>(slot_of), add_big);
            __syncthreads();
            if (tid == 0) {
                uint64_t c[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) c[j] = ((uint64_t)big[2 * j + 1] << 32) | big[2 * j];
                uint64_t w = decide_word(d, cnt[wk] & 0xFFFFu, cnt[wk] >> 16, c);
                if (d.ts + wk == d.total_words - 1) w &= d.last_mask;
                d.out[d.ts - d.out_first + wk] = w;
                pc += __popcll(w);
                slot_of[wk] = kNoSlot;
            }
            __syncthreads();
            base += 1;
            continue;
        }
        for (uint32_t u = tid; u < nb; u += NT) {
            const uint16_t wk = undecided[base + u];
            slot_word[u] = wk;
            slot_of[wk] = (uint16_t)u;
        }
        __syncthreads();
        auto add_entry = [&](uint16_t u, const uint64_t *p) {
            entries[soff[u] + atomicAdd(&sfill[u], 1u)] = reinterpret_cast<uint64_t>(p);
        };
        count_bits(static_cast<const uint16_t *>(slot_of), add_entry);
        __syncthreads();
        if (nb <= (uint32_t)(NT / 32)) {
            // few undecided words (a high threshold's typical tile): a warp per word, the
            // lanes loading its literal words 32 at a time and counting each bit position
            // with a ballot, so the loads are not serialised in one thread
            if ((uint32_t)warp < nb) {
                const uint32_t u = (uint32_t)warp;
                const uint16_t wk = slot_word[u];
                const uint32_t ones = cnt[wk] & 0xFFFFu, dirty = cnt[wk] >> 16;
                const uint64_t *lits = entries + soff[u];
                uint32_t c_lo = 0, c_hi = 0;  // counts of bit `lane` and bit `lane + 32`
                for (uint32_t b0 = 0; b0 < dirty; b0 += 32) {
                    const uint64_t x = b0 + lane < dirty ? *reinterpret_cast<const uint64_t *>(lits[b0 + lane]) : 0ull;
#pragma unroll
                    for (int bit = 0; bit < 32; ++bit) {
                        const uint32_t m_lo = __ballot_sync(0xffffffffu, (x >> bit) & 1u);
                        const uint32_t m_hi = __ballot_sync(0xffffffffu, (x >> (bit + 32)) & 1u);
                        if (lane == bit) {
                            c_lo += __popc(m_lo);
                            c_hi += __popc(m_hi);
                        }
                    }
                }
                const uint32_t lo = __ballot_sync(0xffffffffu, accept_at(d.accept_bits, ones + c_lo));
                const uint32_t hi = __ballot_sync(0xffffffffu, accept_at(d.accept_bits, ones + c_hi));
                if (lane == 0) {
                    uint64_t w = ((uint64_t)hi << 32) | lo;
                    if (d.ts + wk == d.total_words - 1) w &= d.last_mask;
                    d.out[d.ts - d.out_first + wk] = w;
                    pc += __popcll(w);
                    slot_of[wk] = kNoSlot;
                }
            }
            __syncthreads();
            base += nb;
            continue;
        }
        for (uint32_t u = tid; u < nb; u += NT) {
            const uint16_t wk = slot_word[u];
            const uint32_t ones = cnt[wk] & 0xFFFFu, dirty = cnt[wk] >> 16;
            uint64_t c[16];
            const uint64_t *lits = entries + soff[u];
            if (dirty < 16) planes_sum<4>(lits, dirty, c);
            else if (dirty < 256) planes_sum<8>(lits, dirty, c);
            else planes_sum<16>(lits, dirty, c);
            uint64_t w = decide_word(d, ones, dirty, c);
            if (d.ts + wk == d.total_words - 1) w &= d.last_mask;
            d.out[d.ts - d.out_first + wk] = w;
            pc += __popcll(w);
            slot_of[wk] = kNoSlot;
        }
        __syncthreads();
        base += nb;
    }
    return pc;
}

}  // namespace bq
