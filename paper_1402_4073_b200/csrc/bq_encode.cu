// Device canonical RLE encoder: words -> the reference's
// marker/literal stream, exactly as RleBuilder / compress produce it
// (bitmaps.py:351-414).
//
// RleBuilder emits one marker per maximal run of equal fill words (all-0 or
// all-1 words), carrying the literal ("dirty") words that follow it; a leading
// dirty run gets a marker with an empty zero fill; trailing words up to
// ceil(r/64) are zero fill.  So with class(w) in {fill0, fill1, dirty} and the
// change points C_0 = 0 < C_1 < ... (positions where the class changes):
//   * change point j of fill class -> marker(bit, run = C_{j+1} - C_j,
//                                           dirty = C_{j+2} - C_{j+1} if class(j+1) is dirty)
//   * change point 0 of dirty class -> marker(0, 0, C_1 - C_0)
// Output offsets are an exclusive scan of (1 + dirty) over the markers.
// Kernels: classify + flag -> compact change points (CUB) -> per-marker sizes
// -> scan (CUB) -> scatter markers and literal words.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bq_internal.h"

namespace bq {

struct WidenFlag {  // u8 flag -> u32, so the run-id scan accumulates in 32 bits
    __host__ __device__ uint32_t operator()(uint8_t f) const { return f; }
};

__device__ __forceinline__ int word_class(const uint64_t *w, uint64_t n_words, uint64_t i) {
    const uint64_t x = i < n_words ? w[i] : 0ull;
    return x == 0ull ? 0 : (x == ~0ull ? 1 : 2);
}

// flags[i] = 1 where the class changes (always at 0)
__global__ void enc_flags_kernel(const uint64_t *w, uint64_t n_words, uint64_t total, uint8_t *flags) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const int c = word_class(w, n_words, i);
        flags[i] = (i == 0 || c != word_class(w, n_words, i - 1)) ? 1 : 0;
    }
}

// For change point j: size of the marker it opens (1 + dirty words), or 0 if it opens none.
__global__ void enc_sizes_kernel(const uint64_t *w, uint64_t n_words, uint64_t total, const uint32_t *cp,
                                 const uint32_t *n_cp, uint32_t *sizes) {
    const uint32_t m = *n_cp;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint64_t p = cp[j];
        const int c = word_class(w, n_words, p);
        const uint64_t q = (j + 1 < m) ? cp[j + 1] : total;  // end of this class run
        uint32_t sz = 0;
        if (c < 2) {
            uint64_t dirty = 0;
            if (j + 1 < m && word_class(w, n_words, q) == 2) dirty = ((j + 2 < m) ? cp[j + 2] : total) - q;
            sz = 1 + (uint32_t)dirty;
        } else if (j == 0) {
            sz = 1 + (uint32_t)(q - p);
        }
        sizes[j] = sz;
    }
}

// One thread per change point: the marker word only (literals: enc_literals_kernel).
__global__ void enc_markers_kernel(const uint64_t *w, uint64_t n_words, uint64_t total, const uint32_t *cp,
                                   const uint32_t *n_cp, const uint32_t *sizes, const uint64_t *offs, uint64_t *out) {
    const uint32_t m = *n_cp;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t sz = sizes[j];
        if (!sz) continue;
        const uint64_t p = cp[j];
        const int c = word_class(w, n_words, p);
        uint64_t bit = 0, run = 0;
        if (c < 2) {
            bit = (uint64_t)c;
            run = ((j + 1 < m) ? cp[j + 1] : total) - p;
        }
        out[offs[j]] = bit | (run << 1) | ((uint64_t)(sz - 1) << 33);  // bitmaps.py:35-36
    }
}

// One thread per word: a literal word i in dirty run k (runid[i] = k + 1) goes right
// after its marker -- marker k - 1 (the fill run before it) or, for a leading dirty
// run, marker 0 -- at offset i - cp[k] within the group.  Coalesced over words, so a
// long literal run costs no more than its bytes.
__global__ void enc_literals_kernel(const uint64_t *w, uint64_t n_words, const uint32_t *runid, const uint32_t *cp,
                                    const uint64_t *offs, uint64_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = w[i];
        if (x == 0ull || x == ~0ull) continue;
        const uint32_t k = runid[i] - 1;
        const uint32_t m = k ? k - 1 : 0;
        out[offs[m] + 1 + (i - cp[k])] = x;
    }
}

}  // namespace bq

using namespace bq;

extern "C" BQ_API int bq_rle_encode_device(const uint64_t *d_words, uint64_t n_words, uint64_t r_bits, uint64_t *d_out,
                                           uint64_t cap, uint64_t *out_len, void *stream) {
    const uint64_t total = word_count(r_bits);
    if (n_words > total) return set_error(BQ_EINPUT, "more words than bit_length allows");
    if (total >= (1ull << 31)) return set_error(BQ_EINPUT, "device encoder supports < 2^31 words; use bq_rle_encode_host");
    if (out_len) *out_len = 0;
    if (total == 0) return BQ_OK;
    if (n_words && !d_words) return set_error(BQ_EINPUT, "d_words is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // scratch: flags (u8), idx iterator output cp (u32), n_cp, sizes (u32), offs (u64), cub temp
    size_t t_sel = 0, t_scan = 0, t_run = 0;
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, t_sel, it, (uint8_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                               (int)total, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t_scan, (uint32_t *)nullptr, (uint64_t *)nullptr, (int)total, s);
    auto wide = thrust::make_transform_iterator((const uint8_t *)nullptr, WidenFlag());
    cub::DeviceScan::InclusiveSum(nullptr, t_run, wide, (uint32_t *)nullptr, (int)total, s);
    const size_t a_flags = (total + 255) & ~(size_t)255;
    const size_t a_cp = ((total * 4) + 255) & ~(size_t)255;
    const size_t a_off = ((total + 1) * 8 + 255) & ~(size_t)255;
    const size_t a_tmp = (std::max(std::max(t_sel, t_scan), t_run) + 255) & ~(size_t)255;
    const size_t bytes = a_flags + 3 * a_cp + a_off + a_tmp + 256;
    char *base = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&base), bytes, s);
    if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync(encoder scratch)");
    uint8_t *flags = reinterpret_cast<uint8_t *>(base);
    uint32_t *cp = reinterpret_cast<uint32_t *>(base + a_flags);
    uint32_t *sizes = reinterpret_cast<uint32_t *>(base + a_flags + a_cp);
    uint32_t *runid = reinterpret_cast<uint32_t *>(base + a_flags + 2 * a_cp);
    uint64_t *offs = reinterpret_cast<uint64_t *>(base + a_flags + 3 * a_cp);
    void *tmp = base + a_flags + 3 * a_cp + a_off;
    uint32_t *n_cp = reinterpret_cast<uint32_t *>(base + bytes - 256);
    int rc = BQ_OK;
    const int threads = 256;
    const unsigned grid = (unsigned)std::min<uint64_t>((total + threads - 1) / threads, (uint64_t)sm_count() * 16);
    uint64_t h_last[2] = {0, 0};
    uint32_t h_ncp = 0;
    do {
        enc_flags_kernel<<<grid, threads, 0, s>>>(d_words, n_words, total, flags);
        size_t t = a_tmp;
        if ((e = cub::DeviceSelect::Flagged(tmp, t, it, flags, cp, n_cp, (int)total, s)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(&h_ncp, n_cp, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        enc_sizes_kernel<<<grid, threads, 0, s>>>(d_words, n_words, total, cp, n_cp, sizes);
        t = a_tmp;  // exclusive scan over exactly the n_cp change points
        if ((e = cub::DeviceScan::ExclusiveSum(tmp, t, sizes, offs, (int)h_ncp, s)) != cudaSuccess) break;
        // encoded length = offs[n_cp - 1] + sizes[n_cp - 1]
        uint32_t last_size = 0;
        if ((e = cudaMemcpyAsync(&h_last[0], offs + (h_ncp - 1), 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(&last_size, sizes + (h_ncp - 1), 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
        const uint64_t len = h_last[0] + last_size;
        if (out_len) *out_len = len;
        if (len > cap) {
            rc = set_error(BQ_ERESOURCE, "encoding needs %llu words, capacity %llu", (unsigned long long)len,
                           (unsigned long long)cap);
            break;
        }
        if (!d_out) {
            rc = set_error(BQ_EINPUT, "d_out is NULL");
            break;
        }
        enc_markers_kernel<<<grid, threads, 0, s>>>(d_words, n_words, total, cp, n_cp, sizes, offs, d_out);
        if (n_words) {  // run id of every word (1-based change-point index), then the literals
            t = a_tmp;
            auto fl = thrust::make_transform_iterator((const uint8_t *)flags, WidenFlag());
            if ((e = cub::DeviceScan::InclusiveSum(tmp, t, fl, runid, (int)n_words, s)) != cudaSuccess) break;
            enc_literals_kernel<<<grid, threads, 0, s>>>(d_words, n_words, runid, cp, offs, d_out);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        e = cudaStreamSynchronize(s);
    } while (0);
    cudaFreeAsync(base, s);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_error(e, "bq_rle_encode_device");
    return BQ_OK;
}
