// Membership tests for the similarity-query front end (
// reference bench/similarity.py:26-58): which dataset bitmaps contain which
// prototype row ids.  The reference calls RleBitmap / UncompressedBitmap.get
// per (bitmap, rid) in Python (bitmaps.py:107-113, :314-325); here one kernel
// answers the whole (bitmaps x rids) matrix -- a word load per pair for
// uncompressed bitmaps, one marker walk per stream for RLE bitmaps.
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "bq_internal.h"

namespace bq {

__global__ void membership_kernel(const uint64_t *const *ptrs, const uint64_t *lens, int m, const uint64_t *rids, int nr,
                                  uint8_t *out) {
    const uint64_t total = (uint64_t)m * nr;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k / nr), j = (int)(k % nr);
        const uint64_t rid = rids[j], w = rid >> 6;
        out[k] = (w < lens[i]) ? (uint8_t)((__ldg(ptrs[i] + w) >> (rid & 63)) & 1) : 0;
    }
}

// One thread per stream walks its markers once, answering the (sorted) rids in order.
__global__ void rle_membership_kernel(const uint64_t *const *ptrs, const uint64_t *lens, int m, const uint64_t *rids,
                                      int nr, uint8_t *out) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
        const uint64_t *p = ptrs[s];
        const uint64_t L = lens[s];
        uint64_t i = 0, pos = 0;  // next marker, word position of its fill
        int j = 0;
        while (j < nr) {
            const uint64_t rid = rids[j], w = rid >> 6;
            uint8_t v;
            if (i >= L) {  // implicit zero tail
                v = 0;
            } else {
                const uint64_t mk = __ldg(p + i);
                const uint64_t run = (mk >> 1) & 0xFFFFFFFFull, dirty = mk >> 33;
                if (w < pos + run) {  // in the fill
                    v = (uint8_t)(mk & 1);
                } else if (w < pos + run + dirty) {  // in the literals
                    const uint64_t lit = i + 1 + (w - pos - run);
                    v = lit < L ? (uint8_t)((__ldg(p + lit) >> (rid & 63)) & 1) : 0;
                } else {  // past this marker's runs: advance to the next marker
                    pos += run + dirty;
                    i += 1 + dirty;
                    continue;
                }
            }
            out[(uint64_t)s * nr + j] = v;
            ++j;
        }
    }
}

}  // namespace bq

using namespace bq;

template <typename Span>
static int membership(const Span *items, int m, const uint64_t *h_rids, int nr, uint8_t *h_out, int device, bool rle) {
    if (m < 0 || nr < 0 || (m && !items) || (nr && !h_rids) || (m && nr && !h_out))
        return set_error(BQ_EINPUT, "NULL argument");
    if (!m || !nr) return BQ_OK;
    for (int j = 1; j < nr && rle; ++j)
        if (h_rids[j] < h_rids[j - 1]) return set_error(BQ_EINPUT, "rids must be ascending");
    DeviceGuard dg;
    int rc = dg.set(device);
    if (rc) return rc;
    std::vector<const uint64_t *> ptrs(m);
    std::vector<uint64_t> lens(m);
    for (int i = 0; i < m; ++i) {
        ptrs[i] = items[i].words;
        lens[i] = items[i].n_words;
    }
    const size_t bytes = (size_t)m * 16 + (size_t)nr * 8 + (size_t)m * nr;
    char *d = nullptr;
    BQ_CUDA_TRY(cudaMalloc(&d, bytes));
    const uint64_t **d_ptrs = reinterpret_cast<const uint64_t **>(d);
    uint64_t *d_lens = reinterpret_cast<uint64_t *>(d + (size_t)m * 8);
    uint64_t *d_rids = reinterpret_cast<uint64_t *>(d + (size_t)m * 16);
    uint8_t *d_out = reinterpret_cast<uint8_t *>(d + (size_t)m * 16 + (size_t)nr * 8);
    cudaError_t e = cudaMemcpy(d_ptrs, ptrs.data(), (size_t)m * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_lens, lens.data(), (size_t)m * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_rids, h_rids, (size_t)nr * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        if (rle)
            rle_membership_kernel<<<(m + 127) / 128, 128>>>(d_ptrs, d_lens, m, d_rids, nr, d_out);
        else
            membership_kernel<<<(unsigned)(((uint64_t)m * nr + 255) / 256 > 4096 ? 4096 : ((uint64_t)m * nr + 255) / 256),
                                256>>>(d_ptrs, d_lens, m, d_rids, nr, d_out);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(h_out, d_out, (size_t)m * nr, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_error(e, "membership");
    return BQ_OK;
}

extern "C" {

BQ_API int bq_membership(const bq_span *bitmaps, int m, const uint64_t *h_rids, int nr, uint8_t *h_out, int device) {
    return membership(bitmaps, m, h_rids, nr, h_out, device, false);
}

BQ_API int bq_rle_membership(const bq_rle_span *streams, int m, const uint64_t *h_rids, int nr, uint8_t *h_out,
                             int device) {
    return membership(streams, m, h_rids, nr, h_out, device, true);
}

}  // extern "C"
