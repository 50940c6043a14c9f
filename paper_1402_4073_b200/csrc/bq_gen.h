// Counter-based benchmark input generator (K5), one source for host and device.
//
// The reference has no generator for BASELINE.json's Bernoulli configs
// (its bench/datagen.py draws fixed-cardinality sets), so this is new.  It is
// integer-only, so the host (C++) and device (CUDA) produce bit-identical
// words for any (seed, bitmap, word) window; tests/golden/kat.json pins it
// against an independent pure-Python statement (tests/golden/make_golden.py).
//
//   key_i            = mix64(mix64(seed ^ K0) + (i + 1) * GAMMA)
//   rand(key, c)     = mix64(key + (c + 1) * GAMMA)            (SplitMix64 stream)
//   bernoulli(q)     : exact P(bit) = q / 2^16 by composing 16 random words,
//                      least significant digit of q first: x = q_k ? x | R_k : x & R_k
//   density_q(i)     = lo + ((mix64(key_i ^ K1) >> 40) * (hi - lo)) >> 24
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BQ_HD __host__ __device__ __forceinline__
#else
#define BQ_HD static inline
#endif

#define BQ_GAMMA 0x9E3779B97F4A7C15ull

BQ_HD uint64_t bq_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

BQ_HD uint64_t bq_bitmap_key(uint64_t seed, uint64_t i) {
    return bq_mix64(bq_mix64(seed ^ 0x5851F42D4C957F2Dull) + (i + 1) * BQ_GAMMA);
}

BQ_HD uint64_t bq_rand(uint64_t key, uint64_t ctr) { return bq_mix64(key + (ctr + 1) * BQ_GAMMA); }

BQ_HD uint64_t bq_bernoulli_word(uint64_t key, uint64_t w, uint32_t q) {
    if (q == 0) return 0;
    if (q >= 65536u) return ~0ull;
    uint64_t x = 0;
    int k0 = 0;
    while (!((q >> k0) & 1)) ++k0;
    for (int k = k0; k < 16; ++k) {
        uint64_t r = bq_rand(key, w * 16 + (uint64_t)k);
        x = ((q >> k) & 1) ? (x | r) : (x & r);
    }
    return x;
}

BQ_HD uint32_t bq_density_q(uint64_t seed, uint64_t i, uint32_t lo, uint32_t hi) {
    uint64_t u = bq_mix64(bq_bitmap_key(seed, i) ^ 0xD1B54A32D192ED03ull) >> 40;
    return lo + (uint32_t)((u * (uint64_t)(hi - lo)) >> 24);
}
