// Read-bandwidth probe (measurement only, not part of libbq): how fast can one B200
// stream 2 GiB of HBM with 128-bit non-allocating loads, for comparison with the
// copy peak in MEASURED_PEAKS.json.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void __launch_bounds__(256) read_kernel(const uint4 *p, size_t n16, unsigned long long *sink, int unroll) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w) : "l"(p + i + 3 * stride));
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= p[i].x ^ p[i].y ^ p[i].z ^ p[i].w;
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    const size_t bytes = 2ull << 30, n16 = bytes / 16;
    uint4 *p;
    unsigned long long *sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(p, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int occ : {4, 8, 16}) {
        for (int w = 0; w < 3; ++w) read_kernel<<<sms * occ, 256>>>(p, n16, sink, 4);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) read_kernel<<<sms * occ, 256>>>(p, n16, sink, 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d x 256: %.1f GB/s read\n", sms * occ, bytes * reps / (ms / 1e3) / 1e9);
    }
    return 0;
}
