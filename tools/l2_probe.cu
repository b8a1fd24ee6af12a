// l2_probe.cu -- L2 read bandwidth on this GPU: coalesced 16-byte loads over
// an L2-resident buffer (24-96 MB, replayed), and the same over a 2 GB
// buffer (HBM).  Also the 4-byte-per-lane, 128-byte-per-warp pattern of the
// match-set scan (one line per warp per load).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd16(const uint4 *__restrict__ p, size_t n16, int reps, uint32_t *out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *out = acc;
}

// warp reads random 128-byte lines (one 4-byte word per lane), like the
// match-set scan's row reads
__global__ void rd_lines(const uint32_t *__restrict__ p, size_t nlines, int iters, uint32_t *out) {
    const int lane = threadIdx.x & 31;
    uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x - lane + 1);
    uint32_t acc = 0;
    for (int k = 0; k < iters; k++) {
        x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
        const size_t line = (x * 0x2545F4914F6CDD1Dull >> 20) % nlines;
        acc ^= __ldg(p + line * 32 + lane);
    }
    if (acc == 0x12345678u) *out = acc;
}

int main() {
    uint32_t *out;
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t mb : {24, 48, 96, 2048}) {
        const size_t bytes = mb << 20;
        uint4 *p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 1, bytes);
        const int reps = mb >= 1024 ? 2 : 40;
        for (int occ : {4, 8}) {
            rd16<<<sms * occ, 256>>>(p, bytes / 16, 1, out);
            cudaEventRecord(a);
            rd16<<<sms * occ, 256>>>(p, bytes / 16, reps, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("rd16   %5zu MB x%2d  blocks/SM %d: %8.1f GB/s\n", mb, reps, occ, bytes * (double)reps / ms / 1e6);
        }
        for (int occ : {4, 8}) {
            const int iters = 2000;
            const size_t nlines = bytes / 128;
            rd_lines<<<sms * occ, 256>>>((const uint32_t *)p, nlines, 10, out);
            cudaEventRecord(a);
            rd_lines<<<sms * occ, 256>>>((const uint32_t *)p, nlines, iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double lines = (double)sms * occ * 8 * iters;
            printf("lines  %5zu MB random 128B lines, blocks/SM %d: %8.1f GB/s\n", mb, occ, lines * 128 / ms / 1e6);
        }
        cudaFree(p);
    }
    return 0;
}
