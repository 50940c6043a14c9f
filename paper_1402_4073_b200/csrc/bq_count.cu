// K1/K2: word-parallel bit-sliced counting over N uncompressed bitmaps (sm_100a).
//
// Output word w depends only on the N input words at index w (the property
// the reference's horizontal evaluator relies on, circuits/programs.py:208-233),
// so each thread owns two adjacent words (one 128-bit load per input) and
// keeps, in registers, a bit-sliced vertical counter c[0..m) per 32-bit lane,
// m = floor(log2 2N) (circuits/core.py:240-242).
//
// Counting is a Harley-Seal carry-save adder tree: every 16 inputs cost 15
// full adders, each two LOP3s (sum 0x96, majority 0xE8), and one ripple add of
// the weight-16 carry into the high counter bits; ~2.3 LOP3 per input per
// lane.  That replaces the reference's interpreted TreeAdd / SSum / SrtCkt /
// CSvCkt / Looped bitmap programs (circuits/bitparallel.py, programs.py) and
// ScanCount's per-bit increments (counters.py:46-67) with the same function.
//
// Epilogues:
//   MODE_OR / MODE_AND : T = 1 / T = N (wide_or / wide_and, bitmaps.py:647-677)
//   MODE_BREAK         : accept[] as accept[0] XOR (count >= b_1) XOR (count >= b_2) ...,
//                        each ">= b" a bit-sliced comparison with a constant (the
//                        comparator of circuits/core.py:210-237); threshold is one breakpoint.
//   MODE_LUT           : accept[count] read per bit from a shared-memory table
//                        (scan_count_symmetric's lookup, counters.py:81-83).
// The result popcount (cardinality, bitmaps.py:102-105) and the index of the
// last nonzero word (the trim of bitmaps.py:66-67) are reduced in the kernel.
//
// The kernel is a persistent grid-stride loop over tiles of 2 x blockDim words
// (512; narrower CTAs for inputs too small to fill the GPU); the
// input pointer table is staged once per CTA in shared memory.  Loads are
// 128-bit, non-allocating in L1 (each byte is read exactly once).
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>

#include "bq_internal.h"

namespace bq {

constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ld_stream(const uint64_t *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

template <bool FULL>
__device__ __forceinline__ uint4 ld_input(const uint64_t *base, uint64_t w, uint64_t len) {
    if (FULL) return ld_stream(base + w);
    uint4 r = make_uint4(0, 0, 0, 0);
    if (w + 1 < len) {
        r = ld_stream(base + w);
    } else if (w < len) {
        uint64_t v = __ldg(base + w);
        r.x = (uint32_t)v;
        r.y = (uint32_t)(v >> 32);
    }
    return r;
}

__device__ __forceinline__ uint32_t lane_of(const uint4 &v, int l) {
    return l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
}

// full adder: l = a ^ b ^ c (LOP3 0x96), h = maj(a, b, c) (LOP3 0xE8)
#define BQ_CSA(h, l, a, b, c)                \
    do {                                     \
        uint32_t u_ = (a) ^ (b);             \
        uint32_t a_ = (a), c_ = (c);         \
        (h) = (a_ & (b)) | (u_ & c_);        \
        (l) = u_ ^ c_;                       \
    } while (0)

// Add one weight-1 vector into counter bits [lo, M).
template <int M>
__device__ __forceinline__ void ripple_add(uint32_t (&c)[M], uint32_t x, int lo) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
        if (j >= lo) {
            uint32_t t = c[j] & x;
            c[j] ^= x;
            x = t;
        }
    }
}

// count >= b for the bit-sliced count c (M bits, per lane), b a runtime constant.
template <int M>
__device__ __forceinline__ uint32_t ge_const(const uint32_t (&c)[M], uint32_t b) {
    if (b >= (1u << M)) return 0u;
    uint32_t gt = 0u, eq = 0xffffffffu;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
        uint32_t tb = 0u - ((b >> j) & 1u);
        gt |= eq & c[j] & ~tb;
        eq &= ~(c[j] ^ tb);
    }
    return gt | eq;
}

template <int M, int MODE>
__device__ __forceinline__ uint32_t epilogue(const uint32_t (&c)[M], const CountArgs &a,
                                             const uint32_t *slut) {
    if (MODE == MODE_BREAK) {
        uint32_t r = a.accept0;
        for (int b = 0; b < a.nbreak; ++b) r ^= ge_const<M>(c, a.breaks[b]);
        return r;
    } else {  // MODE_LUT
        uint32_t r = 0;
#pragma unroll 4
        for (int bit = 0; bit < 32; ++bit) {
            uint32_t cnt = 0;
#pragma unroll
            for (int j = 0; j < M; ++j) cnt |= ((c[j] >> bit) & 1u) << j;
            r |= ((slut[cnt >> 5] >> (cnt & 31)) & 1u) << bit;
        }
        return r;
    }
}

// Evaluate one 2-word column unit starting at window word w.
template <int M, int MODE, bool FULL>
__device__ __forceinline__ void column(const CountArgs &a, const uint64_t *const *tab, uint64_t w,
                                       const uint32_t *slut, uint32_t (&res)[4]) {
    const int n = a.n;
    if (MODE == MODE_OR || MODE == MODE_AND) {
        uint32_t acc[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[l] = (MODE == MODE_OR) ? 0u : 0xffffffffu;
        int i = 0;
        for (; i + 8 <= n; i += 8) {
            uint4 x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                x[k] = ld_input<FULL>(tab[i + k], w, FULL ? 0 : __ldg(a.lens + i + k));
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int l = 0; l < 4; ++l)
                    acc[l] = (MODE == MODE_OR) ? (acc[l] | lane_of(x[k], l)) : (acc[l] & lane_of(x[k], l));
        }
        if (i < n) {  // tail: up to 7 inputs, loads batched
            uint4 x[7];
#pragma unroll
            for (int k = 0; k < 7; ++k)
                x[k] = (i + k < n) ? ld_input<FULL>(tab[i + k], w, FULL ? 0 : __ldg(a.lens + i + k))
                                   : (MODE == MODE_OR ? make_uint4(0u, 0u, 0u, 0u)
                                                      : make_uint4(~0u, ~0u, ~0u, ~0u));
#pragma unroll
            for (int k = 0; k < 7; ++k)
#pragma unroll
                for (int l = 0; l < 4; ++l)
                    acc[l] = (MODE == MODE_OR) ? (acc[l] | lane_of(x[k], l)) : (acc[l] & lane_of(x[k], l));
        }
#pragma unroll
        for (int l = 0; l < 4; ++l) res[l] = acc[l];
        return;
    } else {
        uint32_t c[4][M];
#pragma unroll
        for (int l = 0; l < 4; ++l)
#pragma unroll
            for (int j = 0; j < M; ++j) c[l][j] = 0u;
        int i = 0;
        if constexpr (M >= 5) {
            for (; i + 16 <= n; i += 16) {
                uint4 x[16];
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    x[k] = ld_input<FULL>(tab[i + k], w, FULL ? 0 : __ldg(a.lens + i + k));
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    uint32_t &ones = c[l][0], &twos = c[l][1], &fours = c[l][2], &eights = c[l][3];
                    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
                    BQ_CSA(twosA, ones, ones, lane_of(x[0], l), lane_of(x[1], l));
                    BQ_CSA(twosB, ones, ones, lane_of(x[2], l), lane_of(x[3], l));
                    BQ_CSA(foursA, twos, twos, twosA, twosB);
                    BQ_CSA(twosA, ones, ones, lane_of(x[4], l), lane_of(x[5], l));
                    BQ_CSA(twosB, ones, ones, lane_of(x[6], l), lane_of(x[7], l));
                    BQ_CSA(foursB, twos, twos, twosA, twosB);
                    BQ_CSA(eightsA, fours, fours, foursA, foursB);
                    BQ_CSA(twosA, ones, ones, lane_of(x[8], l), lane_of(x[9], l));
                    BQ_CSA(twosB, ones, ones, lane_of(x[10], l), lane_of(x[11], l));
                    BQ_CSA(foursA, twos, twos, twosA, twosB);
                    BQ_CSA(twosA, ones, ones, lane_of(x[12], l), lane_of(x[13], l));
                    BQ_CSA(twosB, ones, ones, lane_of(x[14], l), lane_of(x[15], l));
                    BQ_CSA(foursB, twos, twos, twosA, twosB);
                    BQ_CSA(eightsB, fours, fours, foursA, foursB);
                    BQ_CSA(sixteens, eights, eights, eightsA, eightsB);
                    ripple_add<M>(c[l], sixteens, 4);
                }
            }
        }
        for (; i < n; i += 8) {  // remaining < 16 inputs (all of them when N < 16): loads batched by 8
            uint4 x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                x[k] = (i + k < n) ? ld_input<FULL>(tab[i + k], w, FULL ? 0 : __ldg(a.lens + i + k))
                                   : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (i + k < n) {
#pragma unroll
                    for (int l = 0; l < 4; ++l) ripple_add<M>(c[l], lane_of(x[k], l), 0);
                }
        }
#pragma unroll
        for (int l = 0; l < 4; ++l) res[l] = epilogue<M, MODE>(c[l], a, slut);
    }
}

template <int M, int MODE, bool SMEM_TABLE>
__global__ void __launch_bounds__(kThreads) count_kernel(const __grid_constant__ CountArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint64_t **stab = reinterpret_cast<const uint64_t **>(smem);
    uint32_t *slut = reinterpret_cast<uint32_t *>(smem + (SMEM_TABLE ? (size_t)a.n * 8 : 0));
    if (SMEM_TABLE)
            for (int i = threadIdx.x; i < a.n; i += blockDim.x) stab[i] = (a.n <= kSmallN) ? a.small_ptrs[i] : a.ptrs[i];
    if (MODE == MODE_LUT) {
        const int lut_words = ((1 << M) + 31) / 32;
        for (int i = threadIdx.x; i < lut_words; i += blockDim.x) slut[i] = a.lut[i];
    }
    __syncthreads();
    const uint64_t *const *tab = SMEM_TABLE ? stab : a.ptrs;

    unsigned long long pc = 0, lnz = 0;
    const uint64_t tile_words = 2ull * blockDim.x;  // kTileWords, or less for small inputs
    const uint64_t ntiles = (a.nwords + tile_words - 1) / tile_words;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t w = tile * tile_words + 2 * threadIdx.x;
        const bool full = (tile + 1) * tile_words <= a.full_words;  // CTA-uniform
        if (w >= a.nwords) continue;
        uint32_t res[4];
        if (full)
            column<M, MODE, true>(a, tab, w, slut, res);
        else
            column<M, MODE, false>(a, tab, w, slut, res);
        uint64_t lo = (uint64_t)res[0] | ((uint64_t)res[1] << 32);
        uint64_t hi = (uint64_t)res[2] | ((uint64_t)res[3] << 32);
        if (w + 1 >= a.nwords - 1) {
            if (w == a.nwords - 1) lo &= a.last_mask;
            if (w + 1 == a.nwords - 1) hi &= a.last_mask;
        }
        if (w + 1 < a.nwords) {
            *reinterpret_cast<ulonglong2 *>(a.out + w) = make_ulonglong2(lo, hi);
            pc += __popcll(lo) + __popcll(hi);
            if (hi) lnz = w + 2;
            else if (lo) lnz = w + 1;
        } else {
            a.out[w] = lo;
            pc += __popcll(lo);
            if (lo) lnz = w + 1;
        }
    }
    // warp reductions, one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pc += __shfl_down_sync(0xffffffffu, pc, o);
        unsigned long long other = __shfl_down_sync(0xffffffffu, lnz, o);
        lnz = other > lnz ? other : lnz;
    }
    if ((threadIdx.x & 31) == 0) {
        if (a.popcnt && pc) atomicAdd(a.popcnt, pc);
        if (a.last_nz && lnz) atomicMax(a.last_nz, lnz);
    }
}

// ---------------------------------------------------------------------------
// host-side dispatch

using KernelFn = void (*)(CountArgs);

template <int M>
static KernelFn pick(int mode, bool smem_table) {
    switch (mode) {
        case MODE_OR:
            return smem_table ? count_kernel<M, MODE_OR, true> : count_kernel<M, MODE_OR, false>;
        case MODE_AND:
            return smem_table ? count_kernel<M, MODE_AND, true> : count_kernel<M, MODE_AND, false>;
        case MODE_BREAK:
            return smem_table ? count_kernel<M, MODE_BREAK, true> : count_kernel<M, MODE_BREAK, false>;
        default:
            return smem_table ? count_kernel<M, MODE_LUT, true> : count_kernel<M, MODE_LUT, false>;
    }
}

static KernelFn pick_kernel(int m, int mode, bool smem_table) {
    // OR / AND do not use the counter; one instantiation serves every N.
    if (mode == MODE_OR || mode == MODE_AND) return pick<1>(mode, smem_table);
    switch (m) {
        case 1: return pick<1>(mode, smem_table);
        case 2: return pick<2>(mode, smem_table);
        case 3: return pick<3>(mode, smem_table);
        case 4: return pick<4>(mode, smem_table);
        case 5: return pick<5>(mode, smem_table);
        case 6: return pick<6>(mode, smem_table);
        case 7: return pick<7>(mode, smem_table);
        case 8: return pick<8>(mode, smem_table);
        case 9: return pick<9>(mode, smem_table);
        case 10: return pick<10>(mode, smem_table);
        case 11: return pick<11>(mode, smem_table);
        case 12: return pick<12>(mode, smem_table);
        case 13: return pick<13>(mode, smem_table);
        case 14: return pick<14>(mode, smem_table);
        case 15: return pick<15>(mode, smem_table);
        case 16: return pick<16>(mode, smem_table);
        default: return nullptr;
    }
}

static int blocks_per_sm(KernelFn fn, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    uint64_t key = (reinterpret_cast<uint64_t>(fn) * 1315423911ull) ^ ((uint64_t)smem << 8) ^ (uint64_t)dev;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, smem) != cudaSuccess || nb < 1) nb = 1;
    cache[key] = nb;
    return nb;
}

int launch_count(const CountArgs &a, int m, int mode, cudaStream_t stream) {
    if (a.nwords == 0) return BQ_OK;
    const bool smem_table = a.n <= kSmemTableMax;
    KernelFn fn = pick_kernel(m, mode, smem_table);
    if (!fn) return set_error(BQ_EINPUT, "counter width %d unsupported (N too large)", m);
    size_t smem = (smem_table ? (size_t)a.n * 8 : 0) + (mode == MODE_LUT ? (size_t)(((1 << m) + 31) / 32) * 4 : 0);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(count_kernel)");
    }
    // small inputs: narrower CTAs so at least ~2 CTAs per SM get work (C1 is 16k words)
    int threads = kThreads;
    while (threads > 64 && (a.nwords + 2ull * threads - 1) / (2ull * threads) < 2ull * (uint64_t)sm_count()) threads >>= 1;
    const uint64_t ntiles = (a.nwords + 2ull * threads - 1) / (2ull * threads);
    uint64_t grid = (uint64_t)sm_count() * (uint64_t)blocks_per_sm(fn, smem) * (kThreads / threads);
    if (grid > ntiles) grid = ntiles;
    fn<<<(unsigned)grid, threads, smem, stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "count_kernel launch");
    return BQ_OK;
}

}  // namespace bq

// ---------------------------------------------------------------------------
// Whole-bitmap set algebra (bitmaps.py:438-476, 598-644) with fused popcount.
namespace bq {

template <int KIND>
__device__ __forceinline__ uint64_t binop(uint64_t x, uint64_t y) {
    if (KIND == 0) return x & y;   // _u_and: zero beyond the shorter operand
    if (KIND == 1) return x | y;   // _u_or: longer tail copied
    if (KIND == 2) return x ^ y;   // _u_xor
    if (KIND == 3) return x & ~y;  // _u_andnot: a's tail copied
    return ~x;                     // _u_not: complement within r
}

__device__ __forceinline__ ulonglong2 ld_stream2(const uint64_t *p) {
    ulonglong2 v;
    asm("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
    return v;
}

// Two words per thread: 128-bit streaming loads and stores over 16-byte-aligned
// operands (the host falls back to word loads otherwise); words past an operand's
// length read as zero; the popcount and last nonzero index are fused.
template <int KIND, bool VEC>
__device__ __forceinline__ void binop_pair(const uint64_t *__restrict__ a, uint64_t na, const uint64_t *__restrict__ b,
                                           uint64_t nb, uint64_t w, ulonglong2 &x, ulonglong2 &y) {
    if (VEC && w + 1 < na) {
        x = ld_stream2(a + w);
    } else {
        x.x = w < na ? __ldg(a + w) : 0ull;
        x.y = w + 1 < na ? __ldg(a + w + 1) : 0ull;
    }
    y = make_ulonglong2(0ull, 0ull);
    if (KIND != 4) {
        if (VEC && w + 1 < nb) {
            y = ld_stream2(b + w);
        } else {
            y.x = w < nb ? __ldg(b + w) : 0ull;
            y.y = w + 1 < nb ? __ldg(b + w + 1) : 0ull;
        }
    }
}

// Two words per thread, four pairs in flight: 128-bit streaming loads and stores
// over 16-byte-aligned operands (the host falls back to word loads otherwise);
// words past an operand's length read as zero; the popcount and last nonzero
// index are fused.
template <int KIND, bool VEC>
__global__ void __launch_bounds__(256) binop_kernel(const uint64_t *__restrict__ a, uint64_t na,
                                                   const uint64_t *__restrict__ b, uint64_t nb, uint64_t nwords,
                                                   uint64_t last_mask, uint64_t *__restrict__ out,
                                                   unsigned long long *popcnt, unsigned long long *last_nz) {
#ifndef BQ_BINOP_U
#define BQ_BINOP_U 2
#endif
    constexpr int U = BQ_BINOP_U;
    unsigned long long pc = 0, lnz = 0;
    const uint64_t npairs = (nwords + 1) / 2;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npairs; p0 += U * stride) {
        ulonglong2 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p0 + u * stride < npairs) binop_pair<KIND, VEC>(a, na, b, nb, 2 * (p0 + u * stride), x[u], y[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t p = p0 + u * stride;
            if (p >= npairs) break;
            const uint64_t w = 2 * p;
            uint64_t r0 = binop<KIND>(x[u].x, y[u].x), r1 = binop<KIND>(x[u].y, y[u].y);
            if (w + 1 < nwords) {
                if (w + 2 == nwords) r1 &= last_mask;
                if (VEC) {
                    *reinterpret_cast<ulonglong2 *>(out + w) = make_ulonglong2(r0, r1);
                } else {
                    out[w] = r0;
                    out[w + 1] = r1;
                }
                pc += __popcll(r0) + __popcll(r1);
                if (r1) lnz = max(lnz, (unsigned long long)(w + 2));
                else if (r0) lnz = max(lnz, (unsigned long long)(w + 1));
            } else {  // the odd last word
                r0 &= last_mask;
                out[w] = r0;
                pc += __popcll(r0);
                if (r0) lnz = max(lnz, (unsigned long long)(w + 1));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pc += __shfl_down_sync(0xffffffffu, pc, o);
        unsigned long long t = __shfl_down_sync(0xffffffffu, lnz, o);
        lnz = t > lnz ? t : lnz;
    }
    if ((threadIdx.x & 31) == 0) {
        if (popcnt && pc) atomicAdd(popcnt, pc);
        if (last_nz && lnz) atomicMax(last_nz, lnz);
    }
}

typedef void (*BinopFn)(const uint64_t *, uint64_t, const uint64_t *, uint64_t, uint64_t, uint64_t, uint64_t *,
                        unsigned long long *, unsigned long long *);

template <bool VEC>
static BinopFn binop_fn(int kind) {
    switch (kind) {
        case 0: return binop_kernel<0, VEC>;
        case 1: return binop_kernel<1, VEC>;
        case 2: return binop_kernel<2, VEC>;
        case 3: return binop_kernel<3, VEC>;
        default: return binop_kernel<4, VEC>;
    }
}

}  // namespace bq

extern "C" BQ_API int bq_binary_op(int kind, const uint64_t *d_a, uint64_t na, const uint64_t *d_b, uint64_t nb,
                                   uint64_t r_bits, uint64_t *d_out, unsigned long long *d_popcnt,
                                   unsigned long long *d_last_nz, void *stream) {
    using namespace bq;
    if (kind < 0 || kind > 4) return set_error(BQ_EINPUT, "unknown operation %d", kind);
    const uint64_t nwords = word_count(r_bits);
    if (na > nwords || (kind != 4 && nb > nwords)) return set_error(BQ_EINPUT, "more words than bit_length allows");
    if ((na && !d_a) || (kind != 4 && nb && !d_b)) return set_error(BQ_EINPUT, "NULL operand");
    if (nwords && !d_out) return set_error(BQ_EINPUT, "d_out is NULL");
    if (!nwords) return BQ_OK;
    const uint64_t last_mask = (r_bits % W) ? ((1ull << (r_bits % W)) - 1) : ~0ull;
    const bool vec = !((reinterpret_cast<uintptr_t>(d_a) | reinterpret_cast<uintptr_t>(d_out) |
                        (kind == 4 ? 0 : reinterpret_cast<uintptr_t>(d_b))) & 15);
    uint64_t grid = ((nwords + 1) / 2 + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    BinopFn fn = vec ? binop_fn<true>(kind) : binop_fn<false>(kind);
    fn<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        d_a, na, kind == 4 ? nullptr : d_b, kind == 4 ? 0 : nb, nwords, last_mask, d_out, d_popcnt, d_last_nz);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "binop_kernel launch");
    return BQ_OK;
}
