// libbq C ABI: query objects, error reporting, the host-buffer streaming path,
// the canonical RLE encoder and the generators.  See include/bq.h.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "bq_gen.h"
#include "bq_internal.h"

namespace bq {

static thread_local std::string g_last_error;

int set_error(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_error(cudaError_t e, const char *what) {
    // Out-of-memory is the reference's budget idiom (counters.py:54-57): ResourceError.
    int code = (e == cudaErrorMemoryAllocation) ? BQ_ERESOURCE : BQ_ECUDA;
    cudaGetLastError();  // clear sticky-free errors
    return set_error(code, "%s: %s", what, cudaGetErrorString(e));
}

int use_device(int device) {
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    }
    return BQ_OK;
}

// Library memory pool (one per device): RLE query directories, tile-sliced layouts
// and their build scratch are large and allocated once per query object; a
// stream-ordered pool that keeps up to kPoolKeep bytes after frees makes the next
// query's allocations cheap instead of remapping gigabytes per query.
constexpr uint64_t kPoolKeep = 16ull << 30;
static cudaMemPool_t device_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[dev] = p;
    }
    return pools[dev];
}

cudaError_t pool_alloc(void **p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = device_pool(dev);
    if (!pool) return cudaMalloc(p, bytes);
    cudaError_t e = cudaMallocFromPoolAsync(p, bytes, pool, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);  // usable from any stream on return
    return e;
}

cudaError_t pool_alloc_on(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = device_pool(dev);
    if (!pool) return cudaMalloc(p, bytes);
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

void pool_free(void *p) {
    if (!p) return;
    if (cudaFreeAsync(p, 0) != cudaSuccess) cudaGetLastError();
}

void StreamUses::note(cudaStream_t s) {
    for (int i = 0; i < n; ++i)
        if (streams[i] == s) {
            cudaEventRecord(events[i], s);
            return;
        }
    if (n == kMax) {
        overflow = true;
        return;
    }
    if (cudaEventCreateWithFlags(&events[n], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        overflow = true;
        return;
    }
    streams[n] = s;
    cudaEventRecord(events[n], s);
    ++n;
}

void StreamUses::release() {
    for (int i = 0; i < n; ++i) cudaEventDestroy(events[i]);
    n = 0;
}

static cudaStream_t free_stream() {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    std::lock_guard<std::mutex> g(mu);
    if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        streams[dev] = 0;
    }
    return streams[dev];
}

void pool_free_after(void *p, const StreamUses &uses) {
    if (!p) return;
    if (uses.overflow) cudaDeviceSynchronize();
    cudaStream_t fs = free_stream();
    for (int i = 0; i < uses.n; ++i) cudaStreamWaitEvent(fs, uses.events[i], 0);
    if (cudaFreeAsync(p, fs) != cudaSuccess) cudaGetLastError();
}

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 1;
    }
    return cache[dev];
}

// ---------------------------------------------------------------------------
// accept-vector planning shared by the uncompressed and RLE paths

struct AcceptPlan {
    int mode;      // MODE_BREAK or MODE_LUT
    int m;         // counter bits actually needed
    uint32_t accept0;
    int nbreak;
    uint32_t breaks[kMaxBreaks];
    std::vector<uint32_t> lut;  // MODE_LUT, 2^m bits
};

// accept[k] for k = count.  If accept is periodic with period 2^j (j < m) the
// counter only needs j bits (parity: j = 1, a wide XOR).  Few changes of value
// -> breakpoint comparators; many -> lookup table.
static void plan_accept(const uint8_t *acc, int n, AcceptPlan &p) {
    int m = counter_bits(n);
    int j_eff = m;
    for (int j = 0; j < m; ++j) {
        uint32_t per = 1u << j;
        bool periodic = true;
        for (int k = (int)per; k <= n && periodic; ++k)
            if ((acc[k] != 0) != (acc[k % per] != 0)) periodic = false;
        if (periodic) {
            j_eff = j;
            break;
        }
    }
    p.accept0 = acc[0] ? 0xffffffffu : 0u;
    if (j_eff == 0) {  // constant function
        p.mode = MODE_BREAK;
        p.m = 1;
        p.nbreak = 0;
        return;
    }
    int limit = (j_eff < m) ? (1 << j_eff) - 1 : n;  // counts the counter can represent that matter
    std::vector<uint32_t> br;
    for (int k = 1; k <= limit; ++k)
        if ((acc[k] != 0) != (acc[k - 1] != 0)) br.push_back((uint32_t)k);
    p.m = j_eff;
    if ((int)br.size() <= kMaxBreaks) {
        p.mode = MODE_BREAK;
        p.nbreak = (int)br.size();
        for (size_t b = 0; b < br.size(); ++b) p.breaks[b] = br[b];
    } else {
        p.mode = MODE_LUT;
        p.nbreak = 0;
        int entries = 1 << j_eff;
        p.lut.assign((entries + 31) / 32, 0u);
        for (int k = 0; k < entries; ++k) {
            bool v = (k <= n) ? (acc[k] != 0) : false;
            if (v) p.lut[k >> 5] |= 1u << (k & 31);
        }
    }
}

}  // namespace bq

using namespace bq;

// ---------------------------------------------------------------------------
// query objects

struct bq_query {
    int device;
    int n;
    int m;
    uint64_t r_bits, w_begin, w_end, nwords, full_words, last_mask;
    const uint64_t **d_ptrs;
    uint64_t *d_lens;
    std::vector<const uint64_t *> h_ptrs;  // host copy (small N: passed by value to the kernel)
    // device LUTs of MODE_LUT symmetric specs, uploaded once per distinct table
    std::map<std::vector<uint32_t>, CachedTable> luts;
    StreamUses uses;  // caller streams that evaluated this query (destroy waits on them)
    std::mutex mu;    // guards luts / uses
};

extern "C" {

BQ_API int bq_version(void) { return 100; }

BQ_API const char *bq_last_error(void) { return g_last_error.c_str(); }

BQ_API int bq_release_cached_memory(void) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = bq::device_pool(dev);
    if (!pool) return BQ_OK;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
    return e == cudaSuccess ? BQ_OK : bq::cuda_error(e, "cudaMemPoolTrimTo");
}

BQ_API int bq_query_create(const bq_span *inputs, int n, uint64_t r_bits, uint64_t w_begin,
                           uint64_t w_end, int device, bq_query **out) {
    if (!out) return set_error(BQ_EINPUT, "out is NULL");
    *out = nullptr;
    if (n < 1) return set_error(BQ_EINPUT, "need at least one input bitmap");
    if (n > BQ_MAX_INPUTS) return set_error(BQ_EINPUT, "%d inputs exceed BQ_MAX_INPUTS=%d", n, BQ_MAX_INPUTS);
    if (!inputs) return set_error(BQ_EINPUT, "inputs is NULL");
    const uint64_t total = word_count(r_bits);
    if (w_end == UINT64_MAX) w_end = total;
    if (w_end > total || w_begin > w_end)
        return set_error(BQ_EINPUT, "word range [%llu, %llu) outside [0, %llu)", (unsigned long long)w_begin,
                         (unsigned long long)w_end, (unsigned long long)total);
    if (w_begin & 1) return set_error(BQ_EINPUT, "w_begin must be even");
    DeviceGuard dg;
    int rc = dg.set(device);
    if (rc) return rc;
    const uint64_t nwords = w_end - w_begin;
    std::vector<const uint64_t *> ptrs(n);
    std::vector<uint64_t> lens(n);
    uint64_t full = nwords;
    for (int i = 0; i < n; ++i) {
        if (inputs[i].n_words > total)  // bitmaps.py:68-69
            return set_error(BQ_EINPUT, "input %d has %llu words, more than bit_length %llu allows", i,
                             (unsigned long long)inputs[i].n_words, (unsigned long long)r_bits);
        uint64_t len = inputs[i].n_words > w_begin ? std::min(inputs[i].n_words - w_begin, nwords) : 0;
        const uint64_t *p = len ? inputs[i].words + w_begin : nullptr;
        if (len && !inputs[i].words) return set_error(BQ_EINPUT, "input %d: NULL words with n_words > 0", i);
        if (len && (reinterpret_cast<uintptr_t>(p) & 15))
            return set_error(BQ_EINPUT, "input %d: device words must be 16-byte aligned", i);
        ptrs[i] = p;
        lens[i] = len;
        full = std::min(full, len);
    }
    bq_query *q = new bq_query();
    q->device = device;
    q->n = n;
    q->m = counter_bits(n);
    q->r_bits = r_bits;
    q->w_begin = w_begin;
    q->w_end = w_end;
    q->nwords = nwords;
    q->full_words = full;
    q->last_mask = (w_end == total && (r_bits % W)) ? ((1ull << (r_bits % W)) - 1) : ~0ull;
    void *buf = nullptr;
    cudaError_t e = pool_alloc(&buf, (size_t)n * 16);
    if (e != cudaSuccess) {
        delete q;
        return cuda_error(e, "cudaMalloc(query table)");
    }
    q->d_ptrs = reinterpret_cast<const uint64_t **>(buf);
    q->d_lens = reinterpret_cast<uint64_t *>(static_cast<char *>(buf) + (size_t)n * 8);
    // the tables are complete before any stream (including non-blocking ones) can use them
    e = cudaMemcpyAsync(q->d_ptrs, ptrs.data(), (size_t)n * 8, cudaMemcpyHostToDevice, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(q->d_lens, lens.data(), (size_t)n * 8, cudaMemcpyHostToDevice, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) {
        pool_free(buf);
        delete q;
        return cuda_error(e, "cudaMemcpy(query table)");
    }
    q->h_ptrs = ptrs;
    *out = q;
    return BQ_OK;
}

BQ_API void bq_query_destroy(bq_query *q) {
    if (!q) return;
    DeviceGuard dg;
    dg.set(q->device);
    pool_free_after(q->d_ptrs, q->uses);  // after the evaluations enqueued so far; no device sync
    for (auto &kv : q->luts) cached_table_free(kv.second, q->uses);
    q->uses.release();
    delete q;
}

BQ_API uint64_t bq_query_out_words(const bq_query *q) { return q ? q->nwords : 0; }

}  // extern "C"

namespace bq {
int query_view(const bq_query *q, const uint64_t *const **ptrs, const uint64_t **lens, int *n, uint64_t *nwords,
               uint64_t *full_words, uint64_t *last_mask, int *device) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    *ptrs = q->d_ptrs;
    *lens = q->d_lens;
    *n = q->n;
    *nwords = q->nwords;
    *full_words = q->full_words;
    *last_mask = q->last_mask;
    *device = q->device;
    return BQ_OK;
}
}  // namespace bq

extern "C" {

static int base_args(bq_query *q, uint64_t *d_out, unsigned long long *d_popcnt,
                     unsigned long long *d_last_nz, CountArgs &a) {
    if (!q) return set_error(BQ_EINPUT, "query is NULL");
    if (q->nwords && !d_out) return set_error(BQ_EINPUT, "d_out is NULL");
    if (reinterpret_cast<uintptr_t>(d_out) & 15) return set_error(BQ_EINPUT, "d_out must be 16-byte aligned");
    memset(&a, 0, sizeof a);
    a.ptrs = q->d_ptrs;
    a.lens = q->d_lens;
    a.n = q->n;
    if (q->n <= kSmallN)
        for (int i = 0; i < q->n; ++i) a.small_ptrs[i] = q->h_ptrs[i];
    a.nwords = q->nwords;
    a.full_words = q->full_words;
    a.last_mask = q->last_mask;
    a.out = d_out;
    a.popcnt = d_popcnt;
    a.last_nz = d_last_nz;
    return BQ_OK;
}

static void note_use(bq_query *q, cudaStream_t s) {
    std::lock_guard<std::mutex> g(q->mu);
    q->uses.note(s);
}

BQ_API int bq_query_threshold(bq_query *q, int t, uint64_t *d_out, unsigned long long *d_popcnt,
                              unsigned long long *d_last_nz, void *stream) {
    CountArgs a;
    int rc = base_args(q, d_out, d_popcnt, d_last_nz, a);
    if (rc) return rc;
    if (t < 1 || t > q->n) return set_error(BQ_EINPUT, "threshold %d outside [1, %d]", t, q->n);  // counters.py:40-43
    DeviceGuard dg;
    if ((rc = dg.set(q->device))) return rc;
    int mode;
    if (t == 1) mode = MODE_OR;
    else if (t == q->n) mode = MODE_AND;
    else {
        mode = MODE_BREAK;
        a.accept0 = 0;
        a.nbreak = 1;
        a.breaks[0] = (uint32_t)t;
    }
    rc = launch_count(a, q->m, mode, static_cast<cudaStream_t>(stream));
    if (rc == BQ_OK) note_use(q, static_cast<cudaStream_t>(stream));
    return rc;
}

BQ_API int bq_query_symmetric(bq_query *q, const uint8_t *h_accept, uint64_t *d_out,
                              unsigned long long *d_popcnt, unsigned long long *d_last_nz, void *stream) {
    CountArgs a;
    int rc = base_args(q, d_out, d_popcnt, d_last_nz, a);
    if (rc) return rc;
    if (!h_accept) return set_error(BQ_EINPUT, "accept vector is NULL");
    DeviceGuard dg;
    if ((rc = dg.set(q->device))) return rc;
    AcceptPlan p;
    plan_accept(h_accept, q->n, p);
    a.accept0 = p.accept0;
    a.nbreak = p.nbreak;
    memcpy(a.breaks, p.breaks, sizeof(uint32_t) * (size_t)p.nbreak);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (p.mode == MODE_LUT) {
        // the table of each distinct spec is uploaded once per query (repeated
        // evaluations: no allocation or copy), complete before any stream reads it
        constexpr size_t kMaxLuts = 64;
        void *d_lut = nullptr;
        bool owned = false;
        {
            std::lock_guard<std::mutex> g(q->mu);
            auto it = q->luts.find(p.lut);
            if (it != q->luts.end()) {
                d_lut = it->second.p;
                cudaError_t e = cached_table_use(it->second, s);  // after its upload, on any stream
                if (e != cudaSuccess) return cuda_error(e, "lut wait");
            } else if (q->luts.size() < kMaxLuts) {
                CachedTable t;
                cudaError_t e = cached_table_upload(t, p.lut.data(), p.lut.size() * 4, s);
                if (e != cudaSuccess) {
                    if (t.p) pool_free(t.p);
                    if (t.ready) cudaEventDestroy(t.ready);
                    return cuda_error(e, "lut upload");
                }
                d_lut = t.p;
                q->luts.emplace(p.lut, t);
            } else {
                owned = true;
            }
        }
        if (owned) {
            cudaError_t e = pool_alloc(&d_lut, p.lut.size() * 4);
            if (e == cudaSuccess) e = cudaMemcpyAsync(d_lut, p.lut.data(), p.lut.size() * 4, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) {
                if (d_lut) pool_free(d_lut);
                return cuda_error(e, "lut upload");
            }
        }
        a.lut = static_cast<const uint32_t *>(d_lut);
        rc = launch_count(a, p.m, MODE_LUT, s);
        if (owned) {
            StreamUses once;
            once.note(s);
            pool_free_after(d_lut, once);
            once.release();
        }
    } else {
        rc = launch_count(a, p.m, MODE_BREAK, s);
    }
    if (rc == BQ_OK) note_use(q, s);
    return rc;
}

BQ_API int bq_threshold_u64(const bq_span *inputs, int n, uint64_t r_bits, int t, uint64_t *d_out,
                            unsigned long long *d_popcnt, void *stream) {
    bq_query *q = nullptr;
    int rc = bq_query_create(inputs, n, r_bits, 0, UINT64_MAX, -1, &q);
    if (rc) return rc;
    rc = bq_query_threshold(q, t, d_out, d_popcnt, nullptr, stream);
    if (rc == BQ_OK) {
        cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) rc = cuda_error(e, "cudaStreamSynchronize");
    }
    bq_query_destroy(q);
    return rc;
}

BQ_API int bq_symmetric_u64(const bq_span *inputs, int n, uint64_t r_bits, const uint8_t *h_accept,
                            uint64_t *d_out, unsigned long long *d_popcnt, void *stream) {
    bq_query *q = nullptr;
    int rc = bq_query_create(inputs, n, r_bits, 0, UINT64_MAX, -1, &q);
    if (rc) return rc;
    rc = bq_query_symmetric(q, h_accept, d_out, d_popcnt, nullptr, stream);
    if (rc == BQ_OK) {
        cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) rc = cuda_error(e, "cudaStreamSynchronize");
    }
    bq_query_destroy(q);
    return rc;
}

// ---------------------------------------------------------------------------
// host-buffer streaming path

namespace {
struct SweepWorkspace {
    int device = -1;
    void *dev = nullptr;
    size_t dev_bytes = 0;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    std::mutex mu;
};
SweepWorkspace g_sweep[64];
}  // namespace

BQ_API int bq_sweep_host(const uint64_t *const *h_inputs, const uint64_t *n_words, int n, uint64_t r_bits,
                         const int *ts, const uint8_t *h_accepts, int nq, uint64_t *const *h_outs,
                         unsigned long long *h_popcnts, int device, uint64_t chunk_words) {
    if (n < 1 || n > BQ_MAX_INPUTS) return set_error(BQ_EINPUT, "bad input count %d", n);
    if (nq < 1) return set_error(BQ_EINPUT, "need at least one query");
    if (!h_inputs || !n_words || !ts || !h_outs) return set_error(BQ_EINPUT, "NULL argument");
    const uint64_t total = word_count(r_bits);
    for (int i = 0; i < n; ++i) {
        if (n_words[i] > total)
            return set_error(BQ_EINPUT, "input %d has more words than bit_length allows", i);
        if (n_words[i] && !h_inputs[i]) return set_error(BQ_EINPUT, "input %d is NULL", i);
    }
    std::vector<AcceptPlan> plans(nq);
    std::vector<int> modes(nq), ms(nq);
    for (int k = 0; k < nq; ++k) {
        if (!h_outs[k] && total) return set_error(BQ_EINPUT, "output %d is NULL", k);
        if (ts[k] > 0) {
            if (ts[k] > n) return set_error(BQ_EINPUT, "threshold %d outside [1, %d]", ts[k], n);
            AcceptPlan &p = plans[k];
            p.accept0 = 0;
            p.nbreak = 1;
            p.breaks[0] = (uint32_t)ts[k];
            p.m = counter_bits(n);
            modes[k] = ts[k] == 1 ? MODE_OR : ts[k] == n ? MODE_AND : MODE_BREAK;
            ms[k] = p.m;
        } else {
            if (!h_accepts) return set_error(BQ_EINPUT, "query %d is symmetric but accepts is NULL", k);
            plan_accept(h_accepts + (size_t)k * (n + 1), n, plans[k]);
            modes[k] = plans[k].mode;
            ms[k] = plans[k].m;
        }
    }
    int dev = device;
    if (dev < 0) cudaGetDevice(&dev);
    DeviceGuard dg;
    int rc = dg.set(dev);
    if (rc) return rc;
    if (dev >= 64) return set_error(BQ_EINPUT, "device ordinal too large");
    SweepWorkspace &ws = g_sweep[dev];
    std::lock_guard<std::mutex> guard(ws.mu);

    // chunking: ~128 MiB of inputs per chunk (measured best on B200 + PCIe Gen5:
    // small enough that the un-overlapped first copy-in / last copy-out are short),
    // a multiple of the 512-word tile
    uint64_t chunk = chunk_words;
    if (chunk == 0) chunk = std::max<uint64_t>(512, ((128ull << 20) / (8ull * (uint64_t)n)) & ~511ull);
    chunk = (chunk + 511) & ~511ull;
    if (chunk > total) chunk = (total + 1) & ~1ull;
    if (chunk == 0) chunk = 2;
    const uint64_t nchunks = total ? (total + chunk - 1) / chunk : 0;

    // LUT tables for symmetric queries, and per-chunk length tables
    size_t lut_words = 0;
    std::vector<size_t> lut_off(nq, 0);
    for (int k = 0; k < nq; ++k)
        if (modes[k] == MODE_LUT) {
            lut_off[k] = lut_words;
            lut_words += plans[k].lut.size();
        }
    const size_t in_buf = (size_t)n * chunk * 8;
    const size_t out_buf = (size_t)nq * chunk * 8;
    const size_t tables = (size_t)2 * n * 8 + (size_t)nchunks * n * 8;
    const size_t need = 2 * in_buf + 2 * out_buf + tables + lut_words * 4 + (size_t)nq * 8 + 4096;
    if (ws.dev_bytes < need) {
        if (ws.dev) cudaFree(ws.dev);
        ws.dev = nullptr;
        ws.dev_bytes = 0;
        BQ_CUDA_TRY(cudaMalloc(&ws.dev, need));
        ws.dev_bytes = need;
    }
    if (!ws.s_in) {
        BQ_CUDA_TRY(cudaStreamCreateWithFlags(&ws.s_in, cudaStreamNonBlocking));
        BQ_CUDA_TRY(cudaStreamCreateWithFlags(&ws.s_comp, cudaStreamNonBlocking));
        BQ_CUDA_TRY(cudaStreamCreateWithFlags(&ws.s_out, cudaStreamNonBlocking));
    }
    char *base = static_cast<char *>(ws.dev);
    uint64_t *d_in[2] = {reinterpret_cast<uint64_t *>(base), reinterpret_cast<uint64_t *>(base + in_buf)};
    uint64_t *d_out[2] = {reinterpret_cast<uint64_t *>(base + 2 * in_buf),
                          reinterpret_cast<uint64_t *>(base + 2 * in_buf + out_buf)};
    char *tp = base + 2 * in_buf + 2 * out_buf;
    const uint64_t **d_ptrs[2] = {reinterpret_cast<const uint64_t **>(tp),
                                  reinterpret_cast<const uint64_t **>(tp + (size_t)n * 8)};
    uint64_t *d_lens = reinterpret_cast<uint64_t *>(tp + (size_t)2 * n * 8);
    uint32_t *d_lut = reinterpret_cast<uint32_t *>(tp + tables);
    unsigned long long *d_pop =
        reinterpret_cast<unsigned long long *>(tp + tables + ((lut_words * 4 + 15) & ~(size_t)15));

    std::vector<const uint64_t *> hp(2 * (size_t)n);
    for (int b = 0; b < 2; ++b)
        for (int i = 0; i < n; ++i) hp[(size_t)b * n + i] = d_in[b] + (size_t)i * chunk;
    std::vector<uint64_t> hl((size_t)nchunks * n);
    std::vector<uint64_t> full(nchunks);
    for (uint64_t c = 0; c < nchunks; ++c) {
        uint64_t w0 = c * chunk, cw = std::min(chunk, total - w0), f = cw;
        for (int i = 0; i < n; ++i) {
            uint64_t len = n_words[i] > w0 ? std::min(n_words[i] - w0, cw) : 0;
            hl[c * n + i] = len;
            f = std::min(f, len);
        }
        full[c] = f;
    }
    BQ_CUDA_TRY(cudaMemcpy(d_ptrs[0], hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
    if (!hl.empty()) BQ_CUDA_TRY(cudaMemcpy(d_lens, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice));
    for (int k = 0; k < nq; ++k)
        if (modes[k] == MODE_LUT)
            BQ_CUDA_TRY(cudaMemcpy(d_lut + lut_off[k], plans[k].lut.data(), plans[k].lut.size() * 4,
                                   cudaMemcpyHostToDevice));
    // pageable copies may return before their DMA lands, and s_comp does not order
    // after the legacy stream: wait for the tables before the kernels read them
    BQ_CUDA_TRY(cudaStreamSynchronize(0));
    BQ_CUDA_TRY(cudaMemsetAsync(d_pop, 0, (size_t)nq * 8, ws.s_comp));

    // rows of one strided host array (the common layout) allow 2-D copies
    bool uniform = n > 1;
    const int64_t host_pitch = n > 1 ? (int64_t)(h_inputs[1] - h_inputs[0]) : 0;
    for (int i = 1; i < n && uniform; ++i)
        uniform = (h_inputs[i] - h_inputs[i - 1]) == host_pitch && host_pitch >= (int64_t)total;
    cudaEvent_t ev_in[2], ev_comp[2], ev_out[2];
    for (int b = 0; b < 2; ++b) {
        cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_comp[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_out[b], cudaEventDisableTiming);
    }
    bool used[2] = {false, false};
    rc = BQ_OK;
    for (uint64_t c = 0; c < nchunks && rc == BQ_OK; ++c) {
        const int b = (int)(c & 1);
        const uint64_t w0 = c * chunk, cw = std::min(chunk, total - w0);
        if (used[b]) cudaStreamWaitEvent(ws.s_in, ev_comp[b], 0);  // inputs of chunk c-2 consumed
        if (uniform && full[c] == std::min(chunk, total - w0)) {
            // equally strided host rows, all full in this chunk: one 2-D copy
            cudaMemcpy2DAsync(d_in[b], chunk * 8, h_inputs[0] + w0, (size_t)host_pitch * 8, full[c] * 8, (size_t)n,
                              cudaMemcpyHostToDevice, ws.s_in);
        } else {
            for (int i = 0; i < n; ++i) {
                uint64_t len = hl[c * n + i];
                if (len)
                    cudaMemcpyAsync(d_in[b] + (size_t)i * chunk, h_inputs[i] + w0, len * 8, cudaMemcpyHostToDevice,
                                    ws.s_in);
            }
        }
        cudaEventRecord(ev_in[b], ws.s_in);
        cudaStreamWaitEvent(ws.s_comp, ev_in[b], 0);
        if (used[b]) cudaStreamWaitEvent(ws.s_comp, ev_out[b], 0);  // outputs of chunk c-2 copied out
        for (int k = 0; k < nq && rc == BQ_OK; ++k) {
            CountArgs a;
            memset(&a, 0, sizeof a);
            a.ptrs = d_ptrs[b];
            a.lens = d_lens + c * n;
            if (n <= kSmallN)
                for (int i = 0; i < n; ++i) a.small_ptrs[i] = hp[(size_t)b * n + i];
            a.n = n;
            a.nwords = cw;
            a.full_words = full[c];
            a.last_mask = (w0 + cw == total && (r_bits % W)) ? ((1ull << (r_bits % W)) - 1) : ~0ull;
            a.out = d_out[b] + (size_t)k * chunk;
            a.popcnt = d_pop + k;
            a.accept0 = plans[k].accept0;
            a.nbreak = plans[k].nbreak;
            memcpy(a.breaks, plans[k].breaks, sizeof(uint32_t) * (size_t)plans[k].nbreak);
            if (modes[k] == MODE_LUT) a.lut = d_lut + lut_off[k];
            rc = launch_count(a, ms[k], modes[k], ws.s_comp);
        }
        cudaEventRecord(ev_comp[b], ws.s_comp);
        cudaStreamWaitEvent(ws.s_out, ev_comp[b], 0);
        for (int k = 0; k < nq; ++k)
            cudaMemcpyAsync(h_outs[k] + w0, d_out[b] + (size_t)k * chunk, cw * 8, cudaMemcpyDeviceToHost, ws.s_out);
        cudaEventRecord(ev_out[b], ws.s_out);
        used[b] = true;
    }
    if (h_popcnts && rc == BQ_OK) {
        cudaMemcpyAsync(h_popcnts, d_pop, (size_t)nq * 8, cudaMemcpyDeviceToHost, ws.s_comp);
    }
    cudaError_t e1 = cudaStreamSynchronize(ws.s_in);
    cudaError_t e2 = cudaStreamSynchronize(ws.s_comp);
    cudaError_t e3 = cudaStreamSynchronize(ws.s_out);
    for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(ev_in[b]);
        cudaEventDestroy(ev_comp[b]);
        cudaEventDestroy(ev_out[b]);
    }
    if (rc) return rc;
    if (e1 != cudaSuccess) return cuda_error(e1, "sweep copy-in");
    if (e2 != cudaSuccess) return cuda_error(e2, "sweep compute");
    if (e3 != cudaSuccess) return cuda_error(e3, "sweep copy-out");
    return BQ_OK;
}

BQ_API void bq_release_workspace(void) {
    for (auto &ws : g_sweep) {
        std::lock_guard<std::mutex> guard(ws.mu);
        if (ws.dev) {
            cudaFree(ws.dev);
            ws.dev = nullptr;
            ws.dev_bytes = 0;
        }
        if (ws.s_in) {
            cudaStreamDestroy(ws.s_in);
            cudaStreamDestroy(ws.s_comp);
            cudaStreamDestroy(ws.s_out);
            ws.s_in = ws.s_comp = ws.s_out = nullptr;
        }
    }
}

// ---------------------------------------------------------------------------
// canonical RLE encoder (RleBuilder, bitmaps.py:351-414)

}  // extern "C"

namespace bq {

static constexpr uint64_t kMaxFillRun = 0xFFFFFFFFull;  // bitmaps.py:31
static constexpr uint64_t kMaxDirty = 0x7FFFFFFFull;    // bitmaps.py:32

class RleEncoder {
   public:
    RleEncoder(uint64_t *out, uint64_t cap) : out_(out), cap_(cap) {}
    void fill(uint64_t bit, uint64_t count) {
        if (!count) return;
        if (!dirty_.empty() || (run_ && bit_ != bit)) flush();
        bit_ = bit;
        run_ += count;
    }
    void word(uint64_t w) {
        if (w == 0) fill(0, 1);
        else if (w == ~0ull) fill(1, 1);
        else dirty_.push_back(w);
    }
    void finish() {
        if (!dirty_.empty() || run_) flush();
    }
    uint64_t length() const { return len_; }
    bool overflow() const { return len_ > cap_; }

   private:
    void emit(uint64_t w) {
        if (len_ < cap_) out_[len_] = w;
        ++len_;
    }
    void flush() {
        uint64_t run = run_, bit = bit_;
        while (run > kMaxFillRun) {
            emit(bit | (kMaxFillRun << 1));
            run -= kMaxFillRun;
        }
        size_t off = 0, nd = dirty_.size();
        while (nd > kMaxDirty) {
            emit(bit | (run << 1) | (kMaxDirty << 33));
            for (uint64_t k = 0; k < kMaxDirty; ++k) emit(dirty_[off + k]);
            off += kMaxDirty;
            nd -= kMaxDirty;
            run = 0;
            bit = 0;
        }
        emit(bit | (run << 1) | ((uint64_t)nd << 33));
        for (size_t k = 0; k < nd; ++k) emit(dirty_[off + k]);
        bit_ = 0;
        run_ = 0;
        dirty_.clear();
    }
    uint64_t *out_;
    uint64_t cap_;
    uint64_t len_ = 0;
    uint64_t bit_ = 0, run_ = 0;
    std::vector<uint64_t> dirty_;
};

}  // namespace bq

extern "C" {

BQ_API int bq_rle_encode_host(const uint64_t *h_words, uint64_t n_words, uint64_t r_bits, uint64_t *h_out,
                              uint64_t cap, uint64_t *out_len) {
    const uint64_t total = word_count(r_bits);
    if (n_words > total) return set_error(BQ_EINPUT, "more words than bit_length allows");
    RleEncoder enc(h_out, cap);
    for (uint64_t k = 0; k < n_words; ++k) enc.word(h_words[k]);
    enc.fill(0, total - n_words);  // bitmaps.py:412-413
    enc.finish();
    if (out_len) *out_len = enc.length();
    if (enc.overflow()) return set_error(BQ_ERESOURCE, "encoding needs %llu words, capacity %llu",
                                         (unsigned long long)enc.length(), (unsigned long long)cap);
    return BQ_OK;
}

// ---------------------------------------------------------------------------
// generators

BQ_API int bq_gen_bernoulli(uint64_t seed, uint32_t bitmap, uint32_t q16, uint64_t w0, uint64_t nw, uint64_t *out,
                            int on_device, void *stream) {
    if (nw && !out) return set_error(BQ_EINPUT, "out is NULL");
    if (!on_device) {
        const uint64_t key = bq_bitmap_key(seed, bitmap);
        for (uint64_t k = 0; k < nw; ++k) out[k] = bq_bernoulli_word(key, w0 + k, q16);
        return BQ_OK;
    }
    return bq_gen_bernoulli_rows(seed, bitmap, 1, &q16, w0, nw, out, nw, stream);
}

BQ_API int bq_gen_bernoulli_rows(uint64_t seed, uint32_t first, int count, const uint32_t *h_q16s, uint64_t w0,
                                 uint64_t nw, uint64_t *d_out, uint64_t pitch_words, void *stream) {
    if (count <= 0 || nw == 0) return BQ_OK;
    if (!h_q16s || !d_out) return set_error(BQ_EINPUT, "NULL argument");
    if (pitch_words < nw && count > 1) return set_error(BQ_EINPUT, "pitch smaller than row length");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void *d_q = nullptr;
    BQ_CUDA_TRY(cudaMallocAsync(&d_q, (size_t)count * 4, s));
    BQ_CUDA_TRY(cudaMemcpyAsync(d_q, h_q16s, (size_t)count * 4, cudaMemcpyHostToDevice, s));
    int rc = launch_gen_rows(seed, first, count, static_cast<const uint32_t *>(d_q), w0, nw, d_out, pitch_words, s);
    cudaFreeAsync(d_q, s);
    return rc;
}

BQ_API uint32_t bq_gen_density_q16(uint64_t seed, uint32_t bitmap, uint32_t lo, uint32_t hi) {
    return bq_density_q(seed, bitmap, lo, hi);
}

// Geometric run lengths L >= 1 with the given mean, by inversion of a 53-bit
// uniform.  Host only: the device never regenerates these streams.
static uint64_t geometric(uint64_t key, uint64_t ctr, double mean) {
    if (mean <= 1.0) return 1;
    uint64_t r = bq_rand(key, ctr);
    double u = ((double)(r >> 11) + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
    double l = floor(log(u) / log1p(-1.0 / mean));
    if (l > 1e18) l = 1e18;
    return 1 + (uint64_t)l;
}

BQ_API int bq_gen_markov_rle(uint64_t seed, uint32_t bitmap, uint64_t r_bits, double mean_one_run,
                             double mean_zero_run, uint64_t *h_out, uint64_t cap, uint64_t *out_len) {
    if (mean_one_run < 1.0 || mean_zero_run < 1.0) return set_error(BQ_EINPUT, "run means must be >= 1");
    const uint64_t key = bq_bitmap_key(seed ^ 0xC4C4C4C4ull, bitmap);
    RleEncoder enc(h_out, cap);
    // stationary start: P(one) = m1 / (m1 + m0)
    const double p1 = mean_one_run / (mean_one_run + mean_zero_run);
    uint64_t bit = ((double)(bq_rand(key, 0) >> 11) * (1.0 / 9007199254740992.0)) < p1 ? 1 : 0;
    uint64_t pos = 0, cur = 0, ctr = 1;
    while (pos < r_bits) {
        uint64_t len = geometric(key, ctr++, bit ? mean_one_run : mean_zero_run);
        if (len > r_bits - pos) len = r_bits - pos;
        while (len) {
            const uint64_t off = pos & 63;
            if (off == 0 && len >= 64) {
                const uint64_t nfull = len >> 6;
                enc.fill(bit, nfull);
                pos += nfull << 6;
                len -= nfull << 6;
                continue;
            }
            const uint64_t k = std::min<uint64_t>(len, 64 - off);
            if (bit) cur |= (k == 64 ? ~0ull : ((1ull << k) - 1)) << off;
            pos += k;
            len -= k;
            if ((pos & 63) == 0) {
                enc.word(cur);
                cur = 0;
            }
        }
        bit ^= 1;
    }
    if (pos & 63) enc.word(cur);
    enc.finish();
    if (out_len) *out_len = enc.length();
    if (enc.overflow()) return set_error(BQ_ERESOURCE, "stream needs %llu words, capacity %llu",
                                         (unsigned long long)enc.length(), (unsigned long long)cap);
    return BQ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// one query sharded by word range over several devices of one process (SURVEY
// §8(e)): each device evaluates its slice; the only exchange is the popcount sum

extern "C" BQ_API int bq_shard_threshold(int ngpu, const int *devices, const bq_span *spans, int n, uint64_t r_bits,
                              const uint64_t *w_begin, const uint64_t *w_end, int t, uint64_t *const *d_outs,
                              unsigned long long *h_popcnt, void *const *streams) {
    if (ngpu < 1 || !devices || !spans || !w_begin || !w_end || !d_outs) return set_error(BQ_EINPUT, "NULL argument");
    if (n < 1 || n > BQ_MAX_INPUTS) return set_error(BQ_EINPUT, "bad input count %d", n);
    const uint64_t total = word_count(r_bits);
    std::vector<bq_query *> qs(ngpu, nullptr);
    std::vector<unsigned long long *> d_pc(ngpu, nullptr);
    int rc = BQ_OK;
    DeviceGuard dg;
    for (int g = 0; g < ngpu && rc == BQ_OK; ++g) {
        if (w_begin[g] > w_end[g] || w_end[g] > total || (w_begin[g] & 1))
            rc = set_error(BQ_EINPUT, "shard %d: bad word range", g);
        if (rc) break;
        // the shard's inputs are local slices: present them as windows of the whole
        // bitmaps (only words >= w_begin are ever read)
        std::vector<bq_span> in(n);
        for (int i = 0; i < n; ++i) {
            const bq_span &sp = spans[(size_t)g * n + i];
            in[i].words = sp.n_words ? sp.words - w_begin[g] : nullptr;
            in[i].n_words = sp.n_words ? w_begin[g] + sp.n_words : 0;
        }
        rc = bq_query_create(in.data(), n, r_bits, w_begin[g], w_end[g], devices[g], &qs[g]);
        if (rc) break;
        if ((rc = dg.set(devices[g]))) break;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&d_pc[g]), 8, streams ? (cudaStream_t)streams[g] : 0);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_pc[g], 0, 8, streams ? (cudaStream_t)streams[g] : 0);
        if (e != cudaSuccess) rc = cuda_error(e, "shard popcount");
        if (rc == BQ_OK) rc = bq_query_threshold(qs[g], t, d_outs[g], d_pc[g], nullptr, streams ? streams[g] : nullptr);
    }
    unsigned long long sum = 0;
    for (int g = 0; g < ngpu; ++g) {  // the all-reduce of the popcount: 8 bytes per device
        if (!qs[g]) continue;
        dg.set(devices[g]);
        cudaStream_t s = streams ? (cudaStream_t)streams[g] : 0;
        unsigned long long v = 0;
        if (d_pc[g]) {
            cudaError_t e = cudaMemcpyAsync(&v, d_pc[g], 8, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess && rc == BQ_OK) rc = cuda_error(e, "shard popcount");
            cudaFreeAsync(d_pc[g], s);
        }
        sum += v;
        bq_query_destroy(qs[g]);
    }
    if (rc == BQ_OK && h_popcnt) *h_popcnt = sum;
    return rc;
}
