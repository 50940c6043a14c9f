// Internal declarations shared by the libbq translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

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
// Makes `device` current for a scope and restores the caller's current device at
// exit, so a call (or a GC-triggered destroy) never changes the device the caller
// -- e.g. torch -- had selected.
struct DeviceGuard {
    int prev = -1;
    int set(int device) {
        if (device < 0) return BQ_OK;
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess) {
            cudaGetLastError();
            cur = -1;
        }
        if (cur == device) return BQ_OK;
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
        prev = cur;
        return BQ_OK;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
// The library's stream-ordered memory pool (query directories, tile-sliced layouts
// and their build scratch): freed blocks are kept for the next query.
cudaError_t pool_alloc(void **p, size_t bytes);
// Free into the pool in legacy-stream order (no host synchronisation): for memory
// that only legacy-stream work (the synchronous builds) has used.
void pool_free(void *p);
// Evaluations on caller streams that a query's memory must outlive: one event per
// stream, re-recorded after each launch; freeing waits on them on a library stream
// instead of synchronising the device.
struct StreamUses {
    static constexpr int kMax = 16;
    cudaStream_t streams[kMax];
    cudaEvent_t events[kMax];
    int n = 0;
    bool overflow = false;  // more streams than tracked: free after a device sync
    void note(cudaStream_t s);
    void release();  // destroys the events (call after the frees were enqueued)
};
// Free `p` once every evaluation noted in `uses` is done, without a host sync.
void pool_free_after(void *p, const StreamUses &uses);
// Stream-ordered: usable on `s` (and on other streams ordered after it) with no host sync.
cudaError_t pool_alloc_on(void **p, size_t bytes, cudaStream_t s);
int sm_count();              // SMs of the current device

// A small immutable device table cached per query (accept / LUT tables).  Uploaded
// on the first consuming stream with no host synchronisation; `ready` marks the
// upload, and evaluations on any stream wait on it (stream-ordered, not host-side).
struct CachedTable {
    void *p = nullptr;
    cudaEvent_t ready = nullptr;
};
inline cudaError_t cached_table_upload(CachedTable &t, const void *host, size_t bytes, cudaStream_t s) {
    cudaError_t e = pool_alloc_on(&t.p, bytes, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(t.p, host, bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(t.ready, s);
    return e;
}
inline cudaError_t cached_table_use(const CachedTable &t, cudaStream_t s) {
    return t.ready ? cudaStreamWaitEvent(s, t.ready, 0) : cudaSuccess;
}
inline void cached_table_free(CachedTable &t, const StreamUses &uses) {
    if (t.p) pool_free_after(t.p, uses);
    if (t.ready) cudaEventDestroy(t.ready);
    t = CachedTable();
}

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

// ---- K4 over the tile-sliced RLE layout (bq_rle_sliced.cu) -------------------
constexpr int kRleTile = 1024;        // output words per K4 tile (and directory granularity)
constexpr uint16_t kNoSlot = 0xFFFF;  // phase C: word has no bit-counter slot

#ifdef __CUDACC__
__device__ __forceinline__ bool accept_at(const uint32_t *bits, uint32_t c) { return (bits[c >> 5] >> (c & 31)) & 1u; }
#endif

// Tile-sliced layout of n RLE streams, derived once per query from the inputs and
// the K3 directory.  Every (tile, stream) slice -- the stream's words
// [1024 t, 1024 t + 1024) -- is re-encoded as what K4s reads, tile-major:
//  - events (phase A): the nonzero updates the slice's markers make to the packed
//    difference array (ones | dirty << 16) at positions inside the tile, coincident
//    updates of neighbouring markers merged: +1 / -1 where a one-fill starts / ends,
//    +1 / -1 << 16 where a literal group starts / ends, +1 - (1 << 16) where a
//    one-fill starts as a literal group ends, -1 + (1 << 16) where a one-fill ends as
//    a literal group starts.  An event is its 10-bit word position, stored as a byte
//    offset (position * 4) in bits 2-11, 12-21 or 22-31 of a 32-bit word; 16-byte
//    vectors hold 12.  Each tile has six lists, one per kind, holding
//    all slices' events of that kind, each padded to whole warp rows (kEvRow events:
//    32 lanes x one vector), padding slots skipped by their index.  Inside a list the
//    events are permuted so that the 32 updates of each shared-memory atomic
//    instruction (event j of the 32 vectors of a row) fall in distinct banks wherever
//    the list allows: phase A adds a warp-uniform constant per event, every update
//    nonzero and bank-conflict free.
//  - literals (phase C): every slice's literal words inside the tile (literal groups
//    clipped to the tile), ordered position-major: the literal words at word p of
//    the tile are [lit_start[p], lit_start[p + 1]) of the tile's literal array, so
//    phase C reads an undecided word's literals contiguously, with no marker
//    decoding.
constexpr int kEvVec = 12;            // events per 16-byte vector (10-bit positions)
constexpr int kEvRow = 32 * kEvVec;   // events per warp row
constexpr int kEvKinds = 6;
// Per-tile metadata of K4s in schedule order (one 64-byte load per CTA, no
// dependent lookup through the tile order).
struct __align__(16) TileMeta {
    uint4 desc[3];   // the tile's list descriptor (tile_desc)
    uint64_t ebase;  // its first event vector (tile_ebase)
    uint32_t tile;   // the tile
    uint32_t pad;
};
struct SlicedLayout {
    void *mem = nullptr;
    const uint64_t *literals = nullptr;   // [sum of tile literal counts]
    const uint32_t *lit_start = nullptr;  // [ntiles][kRleTile + 1] offset of each word's literals in its tile
    const uint64_t *tile_lbase = nullptr; // [ntiles + 1] literal offset of each tile
    const uint4 *events = nullptr;        // [sum of tile vector counts] 12 packed events per vector
    const uint64_t *tile_ebase = nullptr; // [ntiles + 1] vector offset of each tile
    const uint4 *tile_desc = nullptr;     // [3 ntiles] cumulative ends of the six lists in vectors, their real lengths
    const uint32_t *tile_order = nullptr; // [ntiles] tiles by descending reach (max ones + dirty of a word):
                                          // those that can need phase C are scheduled first
    const TileMeta *tile_meta = nullptr;  // [ntiles] metadata of tile_order[i]
    uint64_t bytes = 0;
    uint64_t n_markers = 0, n_literals = 0;  // n_markers: slice markers (statistic; not stored)
    uint64_t n_events = 0;                   // event slots, padding included (kEvVec per 16-byte vector)
};
// tiles [tile0, tile0 + ntiles) of the streams; directory rows are relative to tile0
int build_sliced(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const uint2 *d_dir, int n, uint32_t tile0,
                 uint32_t ntiles, SlicedLayout *out);
void free_sliced(SlicedLayout *l, const StreamUses *uses = nullptr);
struct SlicedEval {
    int n;
    uint64_t total_words;
    uint32_t tile0;   // first tile of the query's range (output word 0 is word tile0 * kRleTile)
    uint32_t ntiles;  // tiles in the range
    uint64_t last_mask;
    const uint32_t *accept_bits;
    const uint32_t *const_until;
    const uint32_t *breaks;  // counts where accept[] changes; nbreak = -1: too many
    int nbreak;
    uint64_t *out;
    unsigned long long *popcnt;
    int debug;              // BQ_RLE_DEBUG: 1 = skip phase A's updates, 2 = also skip its copies
    uint32_t *reach_out;    // layout build only: each tile's reach, no output
};
int launch_sliced(const SlicedLayout &l, const SlicedEval &e, cudaStream_t stream);

// ---- K3: RLE tile directory (bq_rle_dir.cu) -----------------------------------
// Rows [tile0, tile0 + nrows) of dir[row][stream] = (index of the marker covering
// tile boundary row * kRleTile, word where its fill starts), streams validated
// (err_code 1 truncated literal group, 2 coverage beyond total_words, 3 set bits
// >= r; 0 valid; err_stream the first failing stream).  d_scratch: device memory of
// rle_directory_scratch_bytes(lens) bytes.  Synchronous.
int build_rle_directory(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const std::vector<uint64_t> &lens,
                        uint64_t total_words, uint64_t tail_mask, uint32_t tile0, uint32_t nrows, uint2 *d_dir,
                        void *d_scratch, int *err_code, uint64_t *err_stream, const void *h_extra = nullptr,
                        void *d_extra = nullptr, size_t extra_bytes = 0);
// (h_extra: extra_bytes uploaded to d_extra through the same pinned staging, ordered before the kernel)
// device scratch bytes build_rle_directory needs for these stream lengths
size_t rle_directory_scratch_bytes(const std::vector<uint64_t> &lens);

// ---- K8: cdom sweep statistics (bq_rle_stats.cu) ------------------------------
// h_stats[6] = segments, heap_pops, then the dispatch counts or / and / looped / scan
// of thresholds t > 0 (t = 0: symmetric, no dispatch).  Whole-range directory only.
// Synchronous on `s`.
int rle_sweep_stats(const uint64_t *const *d_ptrs, const uint64_t *d_lens, const uint2 *d_dir, int n,
                    uint32_t ntiles, uint64_t total, int t, uint64_t *h_stats, cudaStream_t s);

// ---- K5 generator kernels --------------------------------------------------
int launch_gen_rows(uint64_t seed, uint32_t first, int count, const uint32_t *d_q16s, uint64_t w0,
                    uint64_t nw, uint64_t *d_out, uint64_t pitch, cudaStream_t stream);

}  // namespace bq
