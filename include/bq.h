/*
 * bq.h -- C ABI of libbq.so, the B200 (sm_100a) threshold / symmetric
 * bitmap-query engine.
 *
 * The reference (Kaser & Lemire's `bitquorum`, /root/reference/pkg/src/
 * bitquorum) has no FFI: its operator API for this path is a set of Python
 * callables plus the algorithm registry.  Each entry point below is what a
 * binding of one of those callables calls; the reference interface it
 * replaces is cited per function (paths relative to pkg/src/bitquorum/).
 * The Python binding that mirrors the reference signatures lives in
 * paper_1402_4073_b200/api.py; INTEGRATION.md shows the ctypes stub a
 * maintainer adds to the reference.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers,
 *    "h_" pointers are host pointers.  Streams are cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Bitmaps are arrays of uint64 words, LSB-first (bitmaps.py:5-6, :24-25).
 *    An input may be shorter than ceil(r/64) words; missing words read as 0
 *    (bitmaps.py:57-58).  Output buffers always hold ceil(r/64) words (or the
 *    window length for ranged queries) with bits >= r cleared.
 *  - Device input/output pointers must be 16-byte aligned (cudaMalloc and
 *    torch allocations are).
 *  - Every function returns a status; 0 is success.  The negative codes map
 *    onto the reference exception classes (errors.py:4-25).  The message of
 *    the last failure on the calling thread is returned by bq_last_error().
 *  - No C++ exceptions cross this boundary.  Calls on distinct query objects
 *    are reentrant; a query object may be used from several streams at once.
 */
#ifndef BQ_H
#define BQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BQ_API __attribute__((visibility("default")))

enum {
    BQ_OK = 0,
    BQ_EINPUT = -1,    /* errors.InputError    (errors.py:8-9)   */
    BQ_ERESOURCE = -2, /* errors.ResourceError (errors.py:16-17) */
    BQ_EFORMAT = -3,   /* errors.FormatError   (errors.py:12-13) */
    BQ_ECUDA = -4      /* CUDA runtime failure (no reference analogue) */
};

/* Largest input count N the device counter supports (m = floor(log2 2N) <= 16). */
#define BQ_MAX_INPUTS 65535

/* One uncompressed input: device words and how many of them are present. */
typedef struct bq_span {
    const uint64_t *words; /* device pointer (may be NULL when n_words == 0) */
    uint64_t n_words;      /* trimmed length; words >= n_words read as zero  */
} bq_span;

/* A prepared query over N device-resident inputs: the device pointer table is
 * uploaded once and reused by every threshold / symmetric evaluation, as the
 * reference's RunContext keeps prebuilt programs per (N, T)
 * (bench/competitions.py:91-104).  Opaque. */
typedef struct bq_query bq_query;

/* Library version, e.g. 100 for 0.1.0. */
BQ_API int bq_version(void);

/* Message of the last failing call on this thread ("" if none). */
BQ_API const char *bq_last_error(void);

/* Return the device memory the library keeps cached for later queries (RLE
 * directories, tile-sliced layouts and their build scratch are taken from a
 * stream-ordered pool that retains up to 16 GiB after frees) to the driver.
 * Synchronizes the current device. */
BQ_API int bq_release_cached_memory(void);

/* Prepare a query over inputs[0..n) whose result has bit length r_bits
 * (= max input bit_length, counters.py:51-52).  Computes output words
 * [w_begin, w_end) of the result (w_end = UINT64_MAX means ceil(r/64)); w_begin
 * must be even.  A word-range query is how one GPU evaluates its shard
 * (horizontal fragmentation; programs.py:196-237).
 * device = CUDA ordinal the inputs live on (-1 = current). */
BQ_API int bq_query_create(const bq_span *inputs, int n, uint64_t r_bits, uint64_t w_begin,
                           uint64_t w_end, int device, bq_query **out);
BQ_API void bq_query_destroy(bq_query *q);
BQ_API uint64_t bq_query_out_words(const bq_query *q);

/* Threshold theta(T; B_1..B_N): bit p set iff p is set in >= t inputs.
 * Replaces counters.scan_count (counters.py:46-67), circuits.looped_threshold
 * (circuits/bitparallel.py:16-43), circuits.csv_threshold (:51-129),
 * circuits.execute of TreeAdd/SSum/SrtCkt programs (circuits/programs.py:163-237),
 * CircuitLibrary.threshold (circuits/library.py:124-128) and, for t == 1 / t == n,
 * bitmaps.wide_or / wide_and (bitmaps.py:647-677).
 * d_out: bq_query_out_words(q) words.  d_popcnt (optional): a device uint64 to
 * which the result's popcount is ADDED (cardinality(), bitmaps.py:102-105).
 * d_last_nz (optional): device uint64 receiving max(index+1) over nonzero
 * output words (atomicMax; lets the caller trim as bitmaps.py:66-67 does).
 * 1 <= t <= n, else BQ_EINPUT (counters.py:40-43). */
BQ_API int bq_query_threshold(bq_query *q, int t, uint64_t *d_out, unsigned long long *d_popcnt,
                              unsigned long long *d_last_nz, void *stream);

/* Arbitrary symmetric function: bit p (p < r) set iff accept[count(p)].
 * h_accept: host array of n + 1 bytes (oracle.SymmetricSpec.accept,
 * oracle.py:17-31).  Replaces counters.scan_count_symmetric (counters.py:70-83)
 * and execute() of circuits.build_symmetric programs (circuits/core.py:349-444). */
BQ_API int bq_query_symmetric(bq_query *q, const uint8_t *h_accept, uint64_t *d_out,
                              unsigned long long *d_popcnt, unsigned long long *d_last_nz,
                              void *stream);

/* One-shot forms (create + evaluate + destroy; the table upload is synchronous). */
BQ_API int bq_threshold_u64(const bq_span *inputs, int n, uint64_t r_bits, int t, uint64_t *d_out,
                            unsigned long long *d_popcnt, void *stream);
BQ_API int bq_symmetric_u64(const bq_span *inputs, int n, uint64_t r_bits, const uint8_t *h_accept,
                            uint64_t *d_out, unsigned long long *d_popcnt, void *stream);

/* One threshold query sharded by word range over `ngpu` devices of ONE process
 * (horizontal fragmentation): device g holds words
 * [w_begin[g], w_end[g]) of every input -- spans[g * n + i] are its local slices
 * (device pointers on devices[g], local word counts) -- and writes that part of
 * the result to d_outs[g] (w_end[g] - w_begin[g] words, bits >= r cleared).  The
 * only exchange is the popcount: the shards' counts are summed into *h_popcnt.
 * w_begin[g] must be even.  streams (optional): one per shard.  Synchronous.
 * Multi-process callers create one bq_query per rank over its range instead and
 * all-reduce the popcount (paper_1402_4073_b200/shard.py: NCCL). */
BQ_API int bq_shard_threshold(int ngpu, const int *devices, const bq_span *spans, int n, uint64_t r_bits,
                              const uint64_t *w_begin, const uint64_t *w_end, int t, uint64_t *const *d_outs,
                              unsigned long long *h_popcnt, void *const *streams);

/* ---- host-buffer path (end to end) ----------------------------------------
 * Evaluate nq queries (thresholds ts[k], or, when ts[k] <= 0, the symmetric
 * spec h_accepts + k*(n+1)) over HOST inputs h_inputs[i] (n_words[i] words,
 * pinned memory recommended), writing each result to host h_outs[k]
 * (ceil(r/64) words) and its popcount to h_popcnts[k].  The word range is
 * streamed through the GPU in chunks of chunk_words words (0 = automatic) with
 * copy-in, compute and copy-out overlapped on separate streams, so inputs larger
 * than HBM work (out-of-core waves).  Blocking.  This is what the reference's
 * Python entry points amount to when handed host bitmaps. */
BQ_API int bq_sweep_host(const uint64_t *const *h_inputs, const uint64_t *n_words, int n,
                         uint64_t r_bits, const int *ts, const uint8_t *h_accepts, int nq,
                         uint64_t *const *h_outs, unsigned long long *h_popcnts, int device,
                         uint64_t chunk_words);

/* Free the device workspace and streams bq_sweep_host keeps cached per device. */
BQ_API void bq_release_workspace(void);

/* ---- run-length-compressed inputs (EWAH-style, bitmaps.py:27-40) ---------- */

/* One compressed input stream on the device. */
typedef struct bq_rle_span {
    const uint64_t *words; /* device pointer to marker/literal words */
    uint64_t n_words;      /* stream length in words */
} bq_rle_span;

typedef struct bq_rle_query bq_rle_query;

/* Decode the marker chains of n streams on the device (K3 directory: the
 * marker governing every tile boundary), validating the encoding as
 * RleBitmap.iter_word_segments does (bitmaps.py:196-219): BQ_EFORMAT on a
 * truncated literal group or a stream covering more than ceil(r/64) words.
 * Synchronous.  The directory is reused by every evaluation (inputs are
 * immutable, bitmaps.py:12-13). */
BQ_API int bq_rle_query_create(const bq_rle_span *streams, int n, uint64_t r_bits, int device,
                               bq_rle_query **out);
/* The same over the output word range [w_begin, w_end) only (multi-GPU word
 * range shards): the streams are the whole, replicated inputs;
 * K3 still walks and validates them whole but keeps directory rows for the
 * range's tiles only, and an evaluation writes words w_begin .. w_end - 1 of the
 * result to d_out[0 ..].  w_begin must be a multiple of 1024 words, w_end too
 * unless it is >= ceil(r/64) (clamped to it). */
BQ_API int bq_rle_query_create_range(const bq_rle_span *streams, int n, uint64_t r_bits, uint64_t w_begin,
                                     uint64_t w_end, int device, bq_rle_query **out);
BQ_API void bq_rle_query_destroy(bq_rle_query *q);
/* Output words of one evaluation (w_end - w_begin). */
BQ_API uint64_t bq_rle_query_out_words(const bq_rle_query *q);
/* Device bytes the query owns: the directory plus, once built, the tile-sliced
 * layout (every 1024-word slice of every stream re-encoded as what K4s reads:
 * the nonzero updates its markers make to the tile's difference array, as packed
 * 10-bit positions in six per-tile lists by update kind, and its literal words,
 * position-major per tile; see SlicedLayout in csrc/bq_internal.h).  The layout is
 * built at the second evaluation of a query (BQ_RLE_SLICED: 0 never, 1 at the
 * first evaluation). */
BQ_API uint64_t bq_rle_query_directory_bytes(const bq_rle_query *q);
/* Size of the tile-sliced layout once built (0, 0 before): markers of the
 * re-encoded slices (a statistic; they are not stored) and 64-bit literal words.
 * K4s reads literals only at undecided words. */
BQ_API int bq_rle_query_layout_stats(const bq_rle_query *q, uint64_t *n_markers, uint64_t *n_literals);

/* Difference-array event slots of the tile-sliced layout once built (0 before):
 * 10-bit entries, 12 per 16-byte vector, padded per tile and kind to whole warp
 * rows; phase A of K4s reads every vector once per evaluation (bench.py's
 * roofline counts n_events / 12 * 16 bytes). */
BQ_API int bq_rle_query_layout_events(const bq_rle_query *q, uint64_t *n_events);

/* Threshold / symmetric function over the compressed inputs, output
 * uncompressed (bq_rle_query_out_words(q) words: ceil(r/64), or the query's
 * word range), popcount ADDED to d_popcnt (optional).  Asynchronous on
 * `stream`, except the evaluation that builds the tile-sliced layout, which
 * synchronizes first.  Replaces runmerge.cdom_threshold
 * (runmerge.py:198-241) and runmerge.cdom_symmetric (:244-299): one-fills
 * count for whole tiles of words, zero-fills are skipped, and dirty words are
 * read only where the fills leave the outcome open. */
BQ_API int bq_rle_query_threshold(bq_rle_query *q, int t, uint64_t *d_out,
                                  unsigned long long *d_popcnt, void *stream);
BQ_API int bq_rle_query_symmetric(bq_rle_query *q, const uint8_t *h_accept, uint64_t *d_out,
                                  unsigned long long *d_popcnt, void *stream);

/* The counters runmerge.cdom_threshold / cdom_symmetric put in ``stats``
 * (runmerge.py:237-240, :296-298), recomputed on the device from the merged runs
 * (_merged_runs, :29-56) through the query's tile directory: h_stats[0] =
 * segments, [1] = heap_pops, [2..5] = dirty_segment_solver's dispatch counts
 * or / and / looped / scan (:69-83) for threshold t (t = 0: symmetric, zeros).
 * The query must cover all words (bq_rle_query_create).  Synchronous on
 * `stream`; scratch ~20 bytes per word, freed before returning. */
BQ_API int bq_rle_query_sweep_stats(bq_rle_query *q, int t, uint64_t *h_stats, void *stream);

/* Canonical RLE encoding of host words, RleBuilder rules (bitmaps.py:351-414);
 * used to hand results back as RleBitmap (counters.py:33-37).  Returns
 * BQ_ERESOURCE if cap is too small; *out_len always receives the needed length. */
BQ_API int bq_rle_encode_host(const uint64_t *h_words, uint64_t n_words, uint64_t r_bits,
                              uint64_t *h_out, uint64_t cap, uint64_t *out_len);

/* The same canonical encoding computed on the device (csrc/bq_encode.cu):
 * d_words (n_words valid words of a ceil(r/64)-word bitmap) -> d_out.  The
 * encoding never exceeds ceil(r/64) + 1 words.  Synchronous on `stream`;
 * *out_len receives the encoded length (also when cap is too small:
 * BQ_ERESOURCE).  Requires ceil(r/64) < 2^31. */
BQ_API int bq_rle_encode_device(const uint64_t *d_words, uint64_t n_words, uint64_t r_bits, uint64_t *d_out,
                                uint64_t cap, uint64_t *out_len, void *stream);

/* ---- whole-bitmap set algebra (bitmaps.py:438-476, :598-644) -------------
 * kind: 0 and, 1 or, 2 xor, 3 andnot (a & ~b), 4 not (~a within r_bits; b unused).
 * Operands of na / nb words (missing words zero); output ceil(r/64) words with
 * bits >= r cleared, popcount ADDED to d_popcnt, max(index+1) of nonzero words
 * to d_last_nz (both optional).  Asynchronous on stream. */
BQ_API int bq_binary_op(int kind, const uint64_t *d_a, uint64_t na, const uint64_t *d_b, uint64_t nb,
                        uint64_t r_bits, uint64_t *d_out, unsigned long long *d_popcnt,
                        unsigned long long *d_last_nz, void *stream);

/* ---- similarity-query front end (bench/similarity.py:26-58) ---------------
 * h_out[i * nr + j] = bit h_rids[j] of bitmap i (UncompressedBitmap.get /
 * RleBitmap.get, bitmaps.py:107-113, :314-325); positions past a bitmap's
 * words read 0.  The RLE form walks each stream once and needs ascending rids.
 * Synchronous. */
BQ_API int bq_membership(const bq_span *bitmaps, int m, const uint64_t *h_rids, int nr, uint8_t *h_out, int device);
BQ_API int bq_rle_membership(const bq_rle_span *streams, int m, const uint64_t *h_rids, int nr, uint8_t *h_out,
                             int device);

/* ---- straight-line BitPrograms (circuits/programs.py) --------------------- */

/* A reference BitProgram (programs.py:56-72) JIT-compiled for sm_100a with
 * NVRTC: one thread per output word, every slot a register.  instr holds
 * n_instr (opcode, dst, a, b) quadruples with the reference opcodes
 * (programs.py:21-28: 0 zero, 1 one, 2 and, 3 or, 4 xor, 5 andnot, 6 not,
 * 7 reclaim).  BQ_EFORMAT for an unknown opcode or slot out of range;
 * BQ_ECUDA if NVRTC / the driver is unavailable.  Opaque. */
typedef struct bq_program bq_program;
BQ_API int bq_program_compile(const int32_t *instr, int n_instr, int arity, int n_slots, int result_slot,
                              bq_program **out);
BQ_API void bq_program_destroy(bq_program *p);
/* The generated CUDA source (NUL-terminated; *len includes the NUL): the GPU
 * counterpart of emit_source (programs.py:332-352). */
BQ_API int bq_program_source(const bq_program *p, char *buf, uint64_t cap, uint64_t *len);
/* Run the program over the inputs of a prepared query (its arity must equal
 * the query's n, programs.py:240-242), like execute / execute_horizontal
 * (programs.py:163-237).  Output and popcount / last-nonzero conventions are
 * those of bq_query_threshold.  Asynchronous on stream. */
BQ_API int bq_program_execute(bq_program *p, bq_query *q, uint64_t *d_out, unsigned long long *d_popcnt,
                              unsigned long long *d_last_nz, void *stream);

/* ---- benchmark input generation (K5, csrc/bq_gen.h) ---------------------- */

/* Words [w0, w0 + nw) of bitmap `bitmap` under `seed`, each bit Bernoulli(q16 / 65536).
 * on_device != 0: out is a device pointer and the words are generated by a kernel
 * on `stream`; otherwise out is host memory. */
BQ_API int bq_gen_bernoulli(uint64_t seed, uint32_t bitmap, uint32_t q16, uint64_t w0, uint64_t nw,
                            uint64_t *out, int on_device, void *stream);
/* Same, for `count` bitmaps laid out with a row pitch (in words) on the device:
 * row i holds bitmap (first + i) with density q16s[i]. */
BQ_API int bq_gen_bernoulli_rows(uint64_t seed, uint32_t first, int count, const uint32_t *h_q16s,
                                 uint64_t w0, uint64_t nw, uint64_t *d_out, uint64_t pitch_words,
                                 void *stream);
/* Quantized per-bitmap density lo + U*(hi-lo) (q16 units). */
BQ_API uint32_t bq_gen_density_q16(uint64_t seed, uint32_t bitmap, uint32_t lo, uint32_t hi);
/* Two-state Markov run generator (host, C4): alternating runs of zeros and ones
 * with geometric lengths of the given means (in bits), encoded canonically.
 * Returns BQ_ERESOURCE if cap is too small (*out_len = needed length). */
BQ_API int bq_gen_markov_rle(uint64_t seed, uint32_t bitmap, uint64_t r_bits, double mean_one_run,
                             double mean_zero_run, uint64_t *h_out, uint64_t cap, uint64_t *out_len);

#ifdef __cplusplus
}
#endif
#endif /* BQ_H */
