// Internal declarations shared by the libbq translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bq.h"

namespace bq {

constexpr int W = 64;

inline uint64_t word_count(uint64_t bits) { return (bits + W - 1) / W; }  // bitmaps.py:43-44

// m = floor(log2(2N)): counter bits needed for counts 0..N (circuits/core.py:240-242).
inline int counter_bits(int n) { return 63 - __builtin_clzll((unsigned long long)(2ull * (uint64_t)n)); }

// ---- error reporting ------------------------------------------------------
int set_error(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int cuda_error(cudaError_t e, const char *what);
#define BQ_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t e_ = (expr);                            \
        if (e_ != cudaSuccess) return ::bq::cuda_error(e_, #expr); \
    } while (0)

int use_device(int device);  // cudaSetDevice when device >= 0
int sm_count();              // SMs of the current device

// ---- K1/K2: uncompressed counting kernel ------------------------------------
constexpr int kMaxBreaks = 32;
constexpr int kMaxCounterBits = 16;
constexpr int kSmemTableMax = 8192;  // pointer tables up to this N live in shared memory
constexpr int kSmallN = 16;          // pointer tables up to this N also travel in the kernel parameters

enum CountMode { MODE_OR = 0, MODE_AND = 1, MODE_BREAK = 2, MODE_LUT = 3 };

struct CountArgs {
    const uint64_t *const *ptrs;  // device table: window start of each input
    const uint64_t *lens;         // device table: valid words of each input in the window
    int n;
    uint64_t nwords;              // output words in the window
    uint64_t full_words;          // every input has >= full_words valid words
    uint64_t last_mask;           // applied to output word nwords - 1
    uint64_t *out;
    unsigned long long *popcnt;   // optional
    unsigned long long *last_nz;  // optional
    uint32_t accept0;             // 0 or 0xffffffff: output at count 0 (before breakpoints)
    int nbreak;
    uint32_t breaks[kMaxBreaks];  // output flips at each count >= breaks[b]
    const uint32_t *lut;          // MODE_LUT: bit-packed accept table, 2^m bits
    const uint64_t *small_ptrs[kSmallN];  // n <= kSmallN: the pointer table by value (no dependent DRAM load)
};

// Launch the counting kernel for counter width m (1..16) and mode.
int launch_count(const CountArgs &a, int m, int mode, cudaStream_t stream);

// ---- K5 generator kernels --------------------------------------------------
int launch_gen_rows(uint64_t seed, uint32_t first, int count, const uint32_t *d_q16s, uint64_t w0,
                    uint64_t nw, uint64_t *d_out, uint64_t pitch, cudaStream_t stream);

}  // namespace bq
