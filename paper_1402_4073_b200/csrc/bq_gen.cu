// K5: device side of the counter-based generator (bq_gen.h) and the host-only
// two-state Markov RLE generator for the compressed config.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "bq_gen.h"
#include "bq_internal.h"

namespace bq {

__global__ void gen_rows_kernel(uint64_t seed, uint32_t first, int count, const uint32_t *q16s,
                                uint64_t w0, uint64_t nw, uint64_t *out, uint64_t pitch) {
    const int row = blockIdx.y;
    if (row >= count) return;
    const uint64_t key = bq_bitmap_key(seed, (uint64_t)first + row);
    const uint32_t q = q16s[row];
    uint64_t *dst = out + (uint64_t)row * pitch;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nw;
         k += (uint64_t)gridDim.x * blockDim.x)
        dst[k] = bq_bernoulli_word(key, w0 + k, q);
}

int launch_gen_rows(uint64_t seed, uint32_t first, int count, const uint32_t *d_q16s, uint64_t w0,
                    uint64_t nw, uint64_t *d_out, uint64_t pitch, cudaStream_t stream) {
    if (count <= 0 || nw == 0) return BQ_OK;
    uint64_t blocks = (nw + 255) / 256;
    uint64_t cap = (uint64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    dim3 grid((unsigned)blocks, (unsigned)count);
    gen_rows_kernel<<<grid, 256, 0, stream>>>(seed, first, count, d_q16s, w0, nw, d_out, pitch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "gen_rows_kernel launch");
    return BQ_OK;
}

}  // namespace bq
