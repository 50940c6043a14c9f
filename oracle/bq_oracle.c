/*
 * oracle/bq_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithms on the threshold /
 * symmetric hot path (Kaser & Lemire, reference package `bitquorum`).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * as the timed CPU baseline.  The product path (paper_1402_4073_b200/) never
 * links or calls it.
 *
 * Parity is pinned against the reference itself: tests/golden/make_golden.py
 * imports the Python reference from /root/reference, runs its algorithms on
 * seeded cases, and commits inputs + outputs as fixtures; tests/test_oracle.py
 * checks every function here against those fixtures.
 *
 * Citations are relative to /root/reference/pkg/src/bitquorum/.
 *
 * Status codes mirror the reference error classes (errors.py:4-25):
 *   0 ok, -1 InputError, -2 ResourceError, -3 FormatError.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINPUT (-1)
#define ORC_ERESOURCE (-2)
#define ORC_EFORMAT (-3)

#define W 64
#define MAX_FILL_RUN 0xFFFFFFFFull  /* bitmaps.py:31 */
#define MAX_DIRTY 0x7FFFFFFFull     /* bitmaps.py:32 */

static inline uint64_t word_count(uint64_t bits) { return (bits + W - 1) / W; } /* bitmaps.py:43-44 */

static inline uint64_t last_mask(uint64_t r) {
    uint64_t rem = r % W;
    return rem ? ((1ull << rem) - 1) : ~0ull;
}

static inline uint64_t in_word(const uint64_t *const *in, const uint64_t *lens, int i, uint64_t w) {
    return w < lens[i] ? in[i][w] : 0; /* missing trailing words read as zero, bitmaps.py:57-58 */
}

/* ---------------------------------------------------------------------------
 * ScanCount (counters.py:46-67): one counter per position, incremented on
 * every set bit, compared with t at the end.  The counters are kept per word
 * (64 at a time) instead of over all r positions; the computation is
 * word-local, so this is the same function with bounded memory.
 */
int orc_scan_count(const uint64_t *const *in, const uint64_t *lens, int n, uint64_t r, int t,
                   uint64_t *out) {
    if (n < 1 || t < 1 || t > n) return ORC_EINPUT; /* counters.py:40-43 */
    uint64_t nw = word_count(r);
    for (uint64_t w = 0; w < nw; ++w) {
        uint32_t counts[W];
        memset(counts, 0, sizeof counts);
        for (int i = 0; i < n; ++i) {
            uint64_t x = in_word(in, lens, i, w);
            while (x) { /* _iter_word_bits, bitmaps.py:47-51 */
                int b = __builtin_ctzll(x);
                counts[b]++;
                x &= x - 1;
            }
        }
        uint64_t o = 0;
        for (int b = 0; b < W; ++b)
            if (counts[b] >= (uint32_t)t) o |= 1ull << b;
        out[w] = o;
    }
    if (nw) out[nw - 1] &= last_mask(r);
    return ORC_OK;
}

/* scan_count_symmetric (counters.py:70-83): output accept[count(p)] for p < r.
 * accept has n + 1 entries (oracle.py:17-31). */
int orc_scan_count_symmetric(const uint64_t *const *in, const uint64_t *lens, int n, uint64_t r,
                             const uint8_t *accept, uint64_t *out) {
    if (n < 1) return ORC_EINPUT;
    uint64_t nw = word_count(r);
    for (uint64_t w = 0; w < nw; ++w) {
        uint32_t counts[W];
        memset(counts, 0, sizeof counts);
        for (int i = 0; i < n; ++i) {
            uint64_t x = in_word(in, lens, i, w);
            while (x) {
                counts[__builtin_ctzll(x)]++;
                x &= x - 1;
            }
        }
        uint64_t o = 0;
        for (int b = 0; b < W; ++b)
            if (accept[counts[b]]) o |= 1ull << b;
        out[w] = o;
    }
    if (nw) out[nw - 1] &= last_mask(r); /* accept[0] sets positions < r only (oracle.py:78-79) */
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * CPU baseline port of the reference's bit-parallel algorithms, evaluated
 * horizontally in word batches (programs.py:196-237 batches of 256 words):
 *   t == 1  -> wide_or   (bitmaps.py:647-663)
 *   t == n  -> wide_and  (bitmaps.py:670-677)
 *   else    -> csv_threshold, the redundant carry-save vertical counter
 *              (circuits/bitparallel.py:51-129), op for op.
 * OpenMP splits the word range across threads (the computation is
 * word-local, programs.py:208-233).
 */
#define BATCH 256
#define MAXM 24

static void csv_batch(const uint64_t *const *in, const uint64_t *lens, int n, int t, uint64_t w0,
                      int width, uint64_t *out) {
    uint64_t c1[MAXM + 1][BATCH], c2[MAXM + 1][BATCH], v[MAXM + 1][BATCH];
    uint64_t carry[BATCH], cin[BATCH], s[BATCH], a[BATCH], b[BATCH];
    int m = 63 - __builtin_clzll((uint64_t)2 * n); /* floor(log2(2N)), bitparallel.py:84 */
    for (int p = 0; p <= m; ++p)
        for (int k = 0; k < width; ++k) c1[p][k] = c2[p][k] = 0;
#define LOAD(dst, i)                                                                  \
    do {                                                                              \
        for (int k = 0; k < width; ++k) dst[k] = in_word(in, lens, (i), w0 + k);      \
    } while (0)
    LOAD(c1[0], 0); /* bitparallel.py:87-88 */
    LOAD(c2[0], 1);
    unsigned time = 1;
    for (int i = 2; i < n; ++i) { /* bitparallel.py:90-100 */
        LOAD(carry, i);
        time += 1;
        int x = __builtin_ctz(time);
        for (int p = 0; p < x; ++p) {
            for (int k = 0; k < width; ++k) {
                uint64_t aa = c1[p][k], bb = c2[p][k];
                uint64_t ss = aa ^ bb;
                c2[p][k] = ss ^ carry[k];
                carry[k] = (aa & bb) | (carry[k] & ss);
                c1[p][k] = 0;
            }
        }
        for (int k = 0; k < width; ++k) c1[x][k] = carry[k];
    }
    /* redundant digits -> binary (bitparallel.py:103-109) */
    for (int k = 0; k < width; ++k) cin[k] = 0;
    for (int p = 0; p <= m; ++p)
        for (int k = 0; k < width; ++k) v[p][k] = 0;
    for (int idx = 0; idx < m; ++idx) {
        for (int k = 0; k < width; ++k) {
            a[k] = c1[idx][k];
            b[k] = c2[idx][k];
            s[k] = a[k] ^ b[k];
            v[idx][k] = s[k] ^ cin[k];
            cin[k] = (a[k] & b[k]) | (cin[k] & s[k]);
        }
    }
    /* subtract t, keep the negated sign (bitparallel.py:112-126) */
    uint64_t minus_t = (1ull << (m + 1)) - (uint64_t)t;
    for (int k = 0; k < width; ++k) cin[k] = 0;
    for (int idx = 0; idx < m; ++idx) {
        if ((minus_t >> idx) & 1)
            for (int k = 0; k < width; ++k) cin[k] |= v[idx][k];
        else
            for (int k = 0; k < width; ++k) cin[k] &= v[idx][k];
    }
    if ((minus_t >> m) & 1)
        for (int k = 0; k < width; ++k) out[k] = v[m][k] ^ cin[k];
    else
        for (int k = 0; k < width; ++k) out[k] = ~(v[m][k] ^ cin[k]);
#undef LOAD
}

int orc_threshold_port(const uint64_t *const *in, const uint64_t *lens, int n, uint64_t r, int t,
                       uint64_t *out, int nthreads) {
    if (n < 1 || t < 1 || t > n) return ORC_EINPUT;
    uint64_t nw = word_count(r);
    int64_t nb = (int64_t)((nw + BATCH - 1) / BATCH);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (int64_t bi = 0; bi < nb; ++bi) {
        uint64_t w0 = (uint64_t)bi * BATCH;
        int width = (int)((nw - w0) < BATCH ? (nw - w0) : BATCH);
        uint64_t *o = out + w0;
        if (t == 1 || t == n) {
            for (int k = 0; k < width; ++k) o[k] = (t == 1) ? 0 : ~0ull;
            for (int i = 0; i < n; ++i) {
                if (t == 1)
                    for (int k = 0; k < width; ++k) o[k] |= in_word(in, lens, i, w0 + k);
                else
                    for (int k = 0; k < width; ++k) o[k] &= in_word(in, lens, i, w0 + k);
            }
        } else {
            csv_batch(in, lens, n, t, w0, width, o);
        }
    }
    if (nw) out[nw - 1] &= last_mask(r);
    return ORC_OK;
}

/* Symmetric CPU baseline: a bit-sliced binary counter (the adder circuits of
 * circuits/core.py:151-207 evaluated horizontally) followed by accept[count]
 * per position, as scan_count_symmetric (counters.py:70-83) decides it. */
int orc_symmetric_port(const uint64_t *const *in, const uint64_t *lens, int n, uint64_t r,
                       const uint8_t *accept, uint64_t *out, int nthreads) {
    if (n < 1) return ORC_EINPUT;
    uint64_t nw = word_count(r);
    int m = 63 - __builtin_clzll((uint64_t)2 * n);
    int64_t nb = (int64_t)((nw + BATCH - 1) / BATCH);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (int64_t bi = 0; bi < nb; ++bi) {
        uint64_t w0 = (uint64_t)bi * BATCH;
        int width = (int)((nw - w0) < BATCH ? (nw - w0) : BATCH);
        uint64_t c[MAXM + 1][BATCH];
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < width; ++k) c[j][k] = 0;
        for (int i = 0; i < n; ++i) {
            for (int k = 0; k < width; ++k) {
                uint64_t carry = in_word(in, lens, i, w0 + k);
                for (int j = 0; j < m && carry; ++j) {
                    uint64_t tt = c[j][k] & carry;
                    c[j][k] ^= carry;
                    carry = tt;
                }
            }
        }
        for (int k = 0; k < width; ++k) {
            uint64_t o = 0;
            for (int bit = 0; bit < W; ++bit) {
                uint32_t cnt = 0;
                for (int j = 0; j < m; ++j) cnt |= (uint32_t)((c[j][k] >> bit) & 1) << j;
                if (accept[cnt]) o |= 1ull << bit;
            }
            out[w0 + k] = o;
        }
    }
    if (nw) out[nw - 1] &= last_mask(r);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * RLE format (bitmaps.py:27-40): marker = fill_bit | run << 1 | dirty << 33,
 * followed by `dirty` literal words; trailing zero fill is implicit.
 */
static inline void split_marker(uint64_t mk, uint64_t *bit, uint64_t *run, uint64_t *dirty) {
    *bit = mk & 1;
    *run = (mk >> 1) & MAX_FILL_RUN;
    *dirty = mk >> 33; /* bitmaps.py:39-40 */
}

/* decompress (bitmaps.py:417-431) over iter_word_segments (:196-219).
 * out has room for word_count(r) words; all of them are written (missing
 * trailing words are zero).  Returns ORC_EFORMAT on the reference's
 * FormatError conditions. */
int orc_rle_decompress(const uint64_t *s, uint64_t len, uint64_t r, uint64_t *out) {
    uint64_t limit = word_count(r);
    uint64_t i = 0, covered = 0;
    while (i < len) {
        uint64_t bit, run, dirty;
        split_marker(s[i], &bit, &run, &dirty);
        i += 1;
        if (run) {
            if (covered + run > limit) return ORC_EFORMAT; /* :426-427 */
            uint64_t f = bit ? ~0ull : 0;
            for (uint64_t k = 0; k < run; ++k) out[covered + k] = f;
            covered += run;
        }
        if (dirty) {
            if (i + dirty > len) return ORC_EFORMAT; /* :210-211 */
            if (covered + dirty > limit) return ORC_EFORMAT;
            memcpy(out + covered, s + i, dirty * 8);
            i += dirty;
            covered += dirty;
        }
    }
    for (uint64_t k = covered; k < limit; ++k) out[k] = 0; /* implicit zero tail, :218-219 */
    /* UncompressedBitmap.__init__ rejects set bits >= r (:70-72) -> FormatError (:428-431) */
    if (limit && (r % W) && (out[limit - 1] & ~last_mask(r))) return ORC_EFORMAT;
    return ORC_OK;
}

/* RleBuilder (bitmaps.py:351-404): canonical encoder. */
typedef struct {
    uint64_t *out;
    uint64_t cap, len;
    uint64_t fill_bit, fill_run;
    uint64_t *dirty;
    uint64_t ndirty, dcap;
    int overflow;
} rle_builder;

static void rb_emit(rle_builder *b, uint64_t w) {
    if (b->len < b->cap)
        b->out[b->len] = w;
    else
        b->overflow = 1;
    b->len++;
}

static void rb_flush(rle_builder *b) { /* bitmaps.py:368-383 */
    uint64_t run = b->fill_run, bit = b->fill_bit;
    while (run > MAX_FILL_RUN) {
        rb_emit(b, bit | (MAX_FILL_RUN << 1));
        run -= MAX_FILL_RUN;
    }
    uint64_t off = 0, nd = b->ndirty;
    while (nd > MAX_DIRTY) {
        rb_emit(b, bit | (run << 1) | (MAX_DIRTY << 33));
        for (uint64_t k = 0; k < MAX_DIRTY; ++k) rb_emit(b, b->dirty[off + k]);
        off += MAX_DIRTY;
        nd -= MAX_DIRTY;
        run = 0;
        bit = 0;
    }
    rb_emit(b, bit | (run << 1) | (nd << 33));
    for (uint64_t k = 0; k < nd; ++k) rb_emit(b, b->dirty[off + k]);
    b->fill_bit = 0;
    b->fill_run = 0;
    b->ndirty = 0;
}

static void rb_append_fill(rle_builder *b, uint64_t bit, uint64_t count) { /* :385-391 */
    if (count == 0) return;
    if (b->ndirty || (b->fill_run && b->fill_bit != bit)) rb_flush(b);
    b->fill_bit = bit;
    b->fill_run += count;
}

static int rb_append_word(rle_builder *b, uint64_t w) { /* :393-399 */
    if (w == 0)
        rb_append_fill(b, 0, 1);
    else if (w == ~0ull)
        rb_append_fill(b, 1, 1);
    else {
        if (b->ndirty == b->dcap) {
            uint64_t nc = b->dcap ? 2 * b->dcap : 1024;
            uint64_t *nd = (uint64_t *)realloc(b->dirty, nc * 8);
            if (!nd) return ORC_ERESOURCE;
            b->dirty = nd;
            b->dcap = nc;
        }
        b->dirty[b->ndirty++] = w;
    }
    return ORC_OK;
}

static void rb_finish(rle_builder *b) { /* :401-404 */
    if (b->ndirty || b->fill_run) rb_flush(b);
}

/* compress (bitmaps.py:407-414).  `words` may be trimmed (nwords <= word_count(r)).
 * On return *out_len holds the encoded length; ORC_ERESOURCE if cap is too small. */
int orc_rle_compress(const uint64_t *words, uint64_t nwords, uint64_t r, uint64_t *out, uint64_t cap,
                     uint64_t *out_len) {
    rle_builder b = {out, cap, 0, 0, 0, NULL, 0, 0, 0};
    int rc = ORC_OK;
    for (uint64_t k = 0; k < nwords && rc == ORC_OK; ++k) rc = rb_append_word(&b, words[k]);
    uint64_t wc = word_count(r);
    if (rc == ORC_OK) {
        rb_append_fill(&b, 0, wc > nwords ? wc - nwords : 0);
        rb_finish(&b);
    }
    free(b.dirty);
    *out_len = b.len;
    if (rc != ORC_OK) return rc;
    return b.overflow ? ORC_ERESOURCE : ORC_OK;
}

/* ---------------------------------------------------------------------------
 * cdom (runmerge.py:198-299): sweep the inputs' merged word runs with a
 * min-heap on run ends.  Output is written uncompressed (word_count(r) words);
 * the reference returns the RleBuilder encoding of exactly these words.
 */
typedef struct {
    const uint64_t *s;
    uint64_t len, i;   /* stream cursor: next marker index */
    uint64_t pos;      /* absolute word position covered so far */
    /* pending segments from the current marker */
    uint64_t f_bit, f_left; /* fill words left */
    uint64_t d_left, d_idx; /* dirty words left, stream index of next literal */
    uint64_t total;
    int err;
} seg_iter;

/* iter_word_segments(total_words) (bitmaps.py:196-219): next raw segment. */
static int seg_next(seg_iter *it, char *kind, uint64_t *x, uint64_t *count) {
    for (;;) {
        if (it->f_left) {
            *kind = 'f';
            *x = it->f_bit;
            *count = it->f_left;
            it->f_left = 0;
            return 1;
        }
        if (it->d_left) {
            *kind = 'd';
            *x = it->d_idx;
            *count = it->d_left;
            it->d_left = 0;
            return 1;
        }
        if (it->i < it->len) {
            uint64_t bit, run, dirty;
            split_marker(it->s[it->i], &bit, &run, &dirty);
            it->i += 1;
            if (dirty && it->i + dirty > it->len) {
                it->err = ORC_EFORMAT;
                return 0;
            }
            it->f_bit = bit;
            it->f_left = run;
            it->d_idx = it->i;
            it->d_left = dirty;
            it->i += dirty;
            it->pos += run + dirty;
            if (it->pos > it->total) {
                it->err = ORC_EFORMAT; /* :216-217 */
                return 0;
            }
            continue;
        }
        if (it->pos < it->total) {
            *kind = 'f';
            *x = 0;
            *count = it->total - it->pos;
            it->pos = it->total;
            return 1;
        }
        return 0;
    }
}

/* _merged_runs (runmerge.py:29-56): adjacent same-bit fills merged. */
typedef struct {
    seg_iter seg;
    int have_pending;
    uint64_t pending_bit, pending_end;
    uint64_t cursor; /* absolute word position */
    int have_look;
    char look_kind;
    uint64_t look_x, look_count;
    int done;
} run_iter;

typedef struct {
    char kind;      /* 'f' or 'd' */
    uint64_t end;   /* inclusive */
    uint64_t bit;   /* fill bit */
    uint64_t base;  /* stream index of the dirty group's first literal */
    uint64_t start; /* absolute word of that literal */
} run_t;

static int run_next(run_iter *ri, run_t *out) {
    for (;;) {
        char kind;
        uint64_t x, count;
        if (ri->done) {
            if (ri->have_pending) {
                out->kind = 'f';
                out->end = ri->pending_end;
                out->bit = ri->pending_bit;
                ri->have_pending = 0;
                return 1;
            }
            return 0;
        }
        if (ri->have_look) {
            kind = ri->look_kind;
            x = ri->look_x;
            count = ri->look_count;
            ri->have_look = 0;
        } else if (!seg_next(&ri->seg, &kind, &x, &count)) {
            ri->done = 1;
            if (ri->seg.err) return 0;
            continue;
        }
        if (kind == 'f') {
            if (ri->have_pending && ri->pending_bit == x) {
                ri->pending_end = ri->cursor + count - 1;
                ri->cursor += count;
                continue;
            }
            if (ri->have_pending) {
                out->kind = 'f';
                out->end = ri->pending_end;
                out->bit = ri->pending_bit;
                ri->pending_bit = x;
                ri->pending_end = ri->cursor + count - 1;
                ri->cursor += count;
                return 1;
            }
            ri->have_pending = 1;
            ri->pending_bit = x;
            ri->pending_end = ri->cursor + count - 1;
            ri->cursor += count;
            continue;
        }
        /* dirty */
        if (ri->have_pending) {
            out->kind = 'f';
            out->end = ri->pending_end;
            out->bit = ri->pending_bit;
            ri->have_pending = 0;
            /* re-deliver this dirty segment next call */
            ri->have_look = 1;
            ri->look_kind = kind;
            ri->look_x = x;
            ri->look_count = count;
            return 1;
        }
        out->kind = 'd';
        out->end = ri->cursor + count - 1;
        out->base = x;
        out->start = ri->cursor;
        ri->cursor += count;
        return 1;
    }
}

typedef struct {
    uint64_t end;
    int idx;
} heap_ent;

static void heap_push(heap_ent *h, int *hn, heap_ent e) {
    int k = (*hn)++;
    while (k > 0) {
        int p = (k - 1) / 2;
        if (h[p].end < e.end || (h[p].end == e.end && h[p].idx <= e.idx)) break;
        h[k] = h[p];
        k = p;
    }
    h[k] = e;
}

static heap_ent heap_pop(heap_ent *h, int *hn) {
    heap_ent top = h[0];
    heap_ent last = h[--(*hn)];
    int k = 0, n = *hn;
    for (;;) {
        int c = 2 * k + 1;
        if (c >= n) break;
        if (c + 1 < n && (h[c + 1].end < h[c].end || (h[c + 1].end == h[c].end && h[c + 1].idx < h[c].idx))) c++;
        if (last.end < h[c].end || (last.end == h[c].end && last.idx <= h[c].idx)) break;
        h[k] = h[c];
        k = c;
    }
    if (n) h[k] = last;
    return top;
}

/* accept == NULL -> threshold t (cdom_threshold); otherwise cdom_symmetric.
 * stats_out (optional, 6 words): segments, heap_pops (runmerge.py:237-239) and the
 * dirty_segment_solver dispatch counts or / and / looped / scan (:69-83; threshold
 * only; cdom_symmetric has no solver). */
static int cdom_common(const uint64_t *const *s, const uint64_t *lens, int n, uint64_t r, int t,
                       const uint8_t *accept, uint64_t *out, uint64_t *stats_out) {
    if (n < 1) return ORC_EINPUT;
    if (!accept && (t < 1 || t > n)) return ORC_EINPUT; /* runmerge.py:201-202 */
    uint64_t total = word_count(r);
    uint64_t rem = r % W;
    if (total == 0) return ORC_OK;
    run_iter *it = (run_iter *)calloc((size_t)n, sizeof(run_iter));
    run_t *cur = (run_t *)calloc((size_t)n, sizeof(run_t));
    heap_ent *heap = (heap_ent *)malloc(sizeof(heap_ent) * (size_t)n);
    int *alive = (int *)calloc((size_t)n, sizeof(int));
    uint32_t (*counts)[W] = NULL;
    int rc = ORC_OK;
    if (!it || !cur || !heap || !alive) {
        rc = ORC_ERESOURCE;
        goto done;
    }
    int hn = 0, ones = 0, clean = 0;
    for (int i = 0; i < n; ++i) { /* _Sweep.__init__, runmerge.py:132-143 */
        it[i].seg.s = s[i];
        it[i].seg.len = lens[i];
        it[i].seg.total = total;
        if (!run_next(&it[i], &cur[i])) {
            rc = it[i].seg.err ? it[i].seg.err : ORC_EFORMAT;
            goto done;
        }
        alive[i] = 1;
        if (cur[i].kind == 'f') {
            clean++;
            ones += (int)cur[i].bit;
        }
        heap_push(heap, &hn, (heap_ent){cur[i].end, i});
    }
    uint64_t pos = 0, segments = 0, pops = 0, br[4] = {0, 0, 0, 0};
    int *dirty_idx = (int *)malloc(sizeof(int) * (size_t)n);
    if (!dirty_idx) {
        rc = ORC_ERESOURCE;
        goto done;
    }
    while (pos < total) { /* runmerge.py:221-236 */
        uint64_t end = heap[0].end;
        segments++;
        int k = ones;
        int dirty_n = n - clean;
        int all_one, all_zero;
        if (!accept) {
            all_one = (t - k <= 0);
            all_zero = (t - k > dirty_n);
        } else { /* runmerge.py:272-276 */
            all_one = 1;
            all_zero = 1;
            for (int c = k; c <= k + dirty_n; ++c) {
                if (accept[c]) all_zero = 0;
                else all_one = 0;
            }
        }
        if (all_one) { /* _emit_ones, runmerge.py:189-195 */
            for (uint64_t w = pos; w <= end; ++w) out[w] = ~0ull;
            if (end == total - 1 && rem) out[end] = (1ull << rem) - 1;
        } else if (all_zero) {
            for (uint64_t w = pos; w <= end; ++w) out[w] = 0;
        } else { /* dirty_segment_solver (:59-126) / per-word count (:277-293) */
            int nd = 0;
            for (int i = 0; i < n; ++i)
                if (alive[i] && cur[i].kind == 'd') dirty_idx[nd++] = i;
            if (!accept) { /* dirty_segment_solver's dispatch (runmerge.py:69-83) */
                const int te = t - k;
                int b;
                if (te == 1) b = 0;
                else if (te == nd) b = 1;
                else if (te >= 128) b = 3; /* SCANCOUNT_CUTOFF */
                else {
                    uint64_t beta = 0;
                    for (int d = 0; d < nd; ++d)
                        for (uint64_t w = pos; w <= end; ++w)
                            beta += (uint64_t)__builtin_popcountll(s[dirty_idx[d]][cur[dirty_idx[d]].base +
                                                                                 (w - cur[dirty_idx[d]].start)]);
                    b = 2 * beta >= (uint64_t)nd * (uint64_t)te ? 2 : 3;
                }
                br[b]++;
            }
            for (uint64_t w = pos; w <= end; ++w) {
                uint32_t cnt[W];
                memset(cnt, 0, sizeof cnt);
                for (int d = 0; d < nd; ++d) {
                    int i = dirty_idx[d];
                    uint64_t x = s[i][cur[i].base + (w - cur[i].start)];
                    while (x) {
                        cnt[__builtin_ctzll(x)]++;
                        x &= x - 1;
                    }
                }
                uint64_t o = 0;
                for (int b = 0; b < W; ++b) {
                    int hit = accept ? accept[k + cnt[b]] : ((int)cnt[b] >= t - k);
                    if (hit) o |= 1ull << b;
                }
                if (w == total - 1 && rem) o &= (1ull << rem) - 1;
                out[w] = o;
            }
        }
        /* _Sweep.advance (:162-177) */
        while (hn && heap[0].end == end) {
            heap_ent e = heap_pop(heap, &hn);
            int i = e.idx;
            pops++;
            if (cur[i].kind == 'f') {
                clean--;
                ones -= (int)cur[i].bit;
            }
            if (run_next(&it[i], &cur[i])) {
                if (cur[i].kind == 'f') {
                    clean++;
                    ones += (int)cur[i].bit;
                }
                heap_push(heap, &hn, (heap_ent){cur[i].end, i});
            } else {
                if (it[i].seg.err) {
                    rc = it[i].seg.err;
                    free(dirty_idx);
                    goto done;
                }
                alive[i] = 0;
                cur[i].kind = 0;
            }
        }
        pos = end + 1;
    }
    free(dirty_idx);
    if (stats_out) {
        stats_out[0] = segments;
        stats_out[1] = pops;
        for (int b = 0; b < 4; ++b) stats_out[2 + b] = br[b];
    }
done:
    free(it);
    free(cur);
    free(heap);
    free(alive);
    free(counts);
    return rc;
}

int orc_cdom_threshold(const uint64_t *const *s, const uint64_t *lens, int n, uint64_t r, int t,
                       uint64_t *out, uint64_t *stats) {
    return cdom_common(s, lens, n, r, t, NULL, out, stats);
}

int orc_cdom_symmetric(const uint64_t *const *s, const uint64_t *lens, int n, uint64_t r,
                       const uint8_t *accept, uint64_t *out, uint64_t *stats) {
    return cdom_common(s, lens, n, r, 0, accept, out, stats);
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Benchmark input generators, restated independently of the product's
 * csrc/bq_gen.h so that bench.py's CPU legs (cpu_baseline, --impl reference)
 * and the tests can build inputs without loading libbq.so.  Pinned by
 * tests/golden/kat.json (Bernoulli / density KATs from an independent
 * pure-Python statement in tests/golden/make_golden.py) and checked equal to
 * the product generator in tests/test_oracle.py.  The reference has no
 * generator for BASELINE.json's configs (its bench/datagen.py draws
 * fixed-cardinality sets), so there is no reference line to cite.
 *
 *   SplitMix64 finaliser; per-bitmap key = mix(mix(seed ^ K0) + (i+1)*GAMMA);
 *   word w of Bernoulli(q/2^16) composes 16 random words, LSB digit of q first.
 */
#include <math.h>

#define ORC_GAMMA 0x9E3779B97F4A7C15ull

static inline uint64_t orc_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t orc_key(uint64_t seed, uint64_t i) {
    return orc_mix(orc_mix(seed ^ 0x5851F42D4C957F2Dull) + (i + 1) * ORC_GAMMA);
}

static inline uint64_t orc_rand(uint64_t key, uint64_t ctr) { return orc_mix(key + (ctr + 1) * ORC_GAMMA); }

static uint64_t orc_bernoulli_word(uint64_t key, uint64_t w, uint32_t q) {
    if (q == 0) return 0;
    if (q >= 65536u) return ~0ull;
    int k0 = __builtin_ctz(q);
    uint64_t x = 0;
    for (int k = k0; k < 16; ++k) {
        uint64_t r = orc_rand(key, w * 16 + (uint64_t)k);
        x = ((q >> k) & 1) ? (x | r) : (x & r);
    }
    return x;
}

/* Words [w0, w0 + nw) of bitmap i, each bit Bernoulli(q16 / 2^16). */
int orc_gen_bernoulli(uint64_t seed, uint32_t bitmap, uint32_t q16, uint64_t w0, uint64_t nw, uint64_t *out) {
    const uint64_t key = orc_key(seed, bitmap);
#pragma omp parallel for schedule(static) if (nw > (1u << 16))
    for (int64_t k = 0; k < (int64_t)nw; ++k) out[k] = orc_bernoulli_word(key, w0 + (uint64_t)k, q16);
    return ORC_OK;
}

/* Per-bitmap density lo + U * (hi - lo) in q16 units (U: 24 bits of the key). */
uint32_t orc_gen_density_q16(uint64_t seed, uint32_t bitmap, uint32_t lo, uint32_t hi) {
    uint64_t u = orc_mix(orc_key(seed, bitmap) ^ 0xD1B54A32D192ED03ull) >> 40;
    return lo + (uint32_t)((u * (uint64_t)(hi - lo)) >> 24);
}

/* Geometric length >= 1 with the given mean, by inverting a 53-bit uniform in (0, 1]. */
static uint64_t orc_geometric(uint64_t key, uint64_t ctr, double mean) {
    if (mean <= 1.0) return 1;
    double u = ((double)(orc_rand(key, ctr) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
    double l = floor(log(u) / log1p(-1.0 / mean));
    if (l > 1e18) l = 1e18;
    return 1 + (uint64_t)l;
}

/* C4 streams: alternating runs of zeros and ones with geometric lengths of the
 * given means (bits), stationary start, encoded canonically with the RleBuilder
 * above (bitmaps.py:351-404).  ORC_ERESOURCE if cap is too small; *out_len is
 * the needed length either way. */
int orc_gen_markov_rle(uint64_t seed, uint32_t bitmap, uint64_t r, double m1, double m0, uint64_t *out,
                       uint64_t cap, uint64_t *out_len) {
    if (m1 < 1.0 || m0 < 1.0) return ORC_EINPUT;
    const uint64_t key = orc_key(seed ^ 0xC4C4C4C4ull, bitmap);
    rle_builder b = {out, cap, 0, 0, 0, NULL, 0, 0, 0};
    const double p1 = m1 / (m1 + m0);
    uint64_t bit = ((double)(orc_rand(key, 0) >> 11) * (1.0 / 9007199254740992.0)) < p1 ? 1 : 0;
    uint64_t pos = 0, cur = 0, ctr = 1;
    int rc = ORC_OK;
    while (pos < r && rc == ORC_OK) {
        uint64_t len = orc_geometric(key, ctr++, bit ? m1 : m0);
        if (len > r - pos) len = r - pos;
        while (len && rc == ORC_OK) {
            uint64_t off = pos & 63;
            if (off == 0 && len >= 64) {
                uint64_t nfull = len >> 6;
                rb_append_fill(&b, bit, nfull);
                pos += nfull << 6;
                len -= nfull << 6;
                continue;
            }
            uint64_t k = len < 64 - off ? len : 64 - off;
            if (bit) cur |= (k == 64 ? ~0ull : ((1ull << k) - 1)) << off;
            pos += k;
            len -= k;
            if ((pos & 63) == 0) {
                rc = rb_append_word(&b, cur);
                cur = 0;
            }
        }
        bit ^= 1;
    }
    if (rc == ORC_OK && (pos & 63)) rc = rb_append_word(&b, cur);
    if (rc == ORC_OK) rb_finish(&b);
    free(b.dirty);
    *out_len = b.len;
    if (rc != ORC_OK) return rc;
    return b.overflow ? ORC_ERESOURCE : ORC_OK;
}
