// Phases B and C shared by the RLE tile kernels K4 (bq_rle.cu) and K4s
// (bq_rle_sliced.cu): one CTA per 1024-word tile, after phase A has built the
// packed difference array cnt[0..1024] (one-fills in bits 0-15, dirty inputs in
// bits 16-31).  This is the decision half of runmerge.cdom_threshold /
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

// Phase C shared memory: [SLOTS][32] packed bit counters | slot_of[kRleTile] | slot_word[SLOTS].
template <int SLOTS>
constexpr size_t tile_resolve_bytes() {
    return (size_t)SLOTS * 128 + (size_t)kRleTile * 2 + (size_t)SLOTS * 2;
}

// Phase C, in batches of SLOTS undecided words: count_bits(slot_of, add_bits) is
// called by every thread between barriers and must call add_bits(slot, word)
// for every literal word whose tile position p has slot_of[p] != kNoSlot.
template <int NT, int SLOTS, class CountBits>
__device__ __forceinline__ unsigned long long tile_resolve(const TileDecide &d, const uint32_t *cnt,
                                                           const uint16_t *undecided, uint32_t nu, uint8_t *region,
                                                           CountBits &&count_bits) {
    const int tid = threadIdx.x;
    uint32_t (*bitcnt)[32] = reinterpret_cast<uint32_t (*)[32]>(region);
    uint16_t *slot_of = reinterpret_cast<uint16_t *>(region + (size_t)SLOTS * 128);
    uint16_t *slot_word = slot_of + kRleTile;
    unsigned long long pc = 0;
    if (!nu) return 0;
    for (int k = tid; k < kRleTile; k += NT) slot_of[k] = kNoSlot;
    __syncthreads();
    auto add_bits = [&](uint16_t u, uint64_t x) {
        while (x) {
            const int b = __ffsll((long long)x) - 1;
            atomicAdd(&bitcnt[u][b & 31], (b < 32) ? 1u : 0x10000u);
            x &= x - 1;
        }
    };
    for (uint32_t base = 0; base < nu; base += SLOTS) {
        const uint32_t nb = min((uint32_t)SLOTS, nu - base);
        for (uint32_t u = tid; u < nb; u += NT) {
            const uint16_t wk = undecided[base + u];
            slot_word[u] = wk;
            slot_of[wk] = (uint16_t)u;
        }
        for (int k = tid; k < SLOTS * 32; k += NT) (&bitcnt[0][0])[k] = 0u;
        __syncthreads();
        count_bits(static_cast<const uint16_t *>(slot_of), add_bits);
        __syncthreads();
        for (uint32_t u = tid; u < nb; u += NT) {
            const uint16_t wk = slot_word[u];
            const uint32_t ones = cnt[wk] & 0xFFFFu;
            uint64_t w = 0;
            for (int b = 0; b < 64; ++b) {
                const uint32_t cb = (bitcnt[u][b & 31] >> ((b >> 5) * 16)) & 0xFFFFu;
                if (accept_at(d.accept_bits, ones + cb)) w |= 1ull << b;
            }
            if (d.ts + wk == d.total_words - 1) w &= d.last_mask;
            d.out[d.ts - d.out_first + wk] = w;
            pc += __popcll(w);
            slot_of[wk] = kNoSlot;
        }
        __syncthreads();
    }
    return pc;
}

}  // namespace bq
